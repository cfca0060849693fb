mkdir -p gpurun_out/r31
for D in 0 1; do for v in 417 414 418; do TNX_GEMM_DPAIR=$D python tools/profile_vertex.py cfg5_syc53_m12 $v >> gpurun_out/r31/d$D.log 2>&1; done; done
TNX_DEBUG_PLAN=1 python tools/profile_vertex.py cfg5_syc53_m12 417 > gpurun_out/r31/plan.log 2>&1
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_northstar.py tests/test_gpu_configs.py -q -m gpu -x > gpurun_out/r31/pytest.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/r31/pytest.log
for D in 0 1; do
  TNX_GEMM_DPAIR=$D timeout 600 python bench.py --config cfg5_syc53_m12 --steps 10 --no-cpu-baseline --no-e2e --sustained-s 0 --secondary "" > gpurun_out/r31/bench5_d$D.json 2>/dev/null
  TNX_GEMM_DPAIR=$D timeout 600 python bench.py --config cfg2_5reg100 --steps 10 --no-cpu-baseline --no-e2e --sustained-s 0 --secondary "" > gpurun_out/r31/bench2_d$D.json 2>/dev/null
  TNX_GEMM_DPAIR=$D timeout 600 python bench.py --steps 20 --no-cpu-baseline --no-e2e --sustained-s 0 --secondary "" > gpurun_out/r31/bench4_d$D.json 2>/dev/null
  echo "d$D"
done
