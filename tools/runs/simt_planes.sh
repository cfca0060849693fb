mkdir -p gpurun_out/r34
timeout 1200 python -m pytest tests -q -m gpu -x > gpurun_out/r34/pytest.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/r34/pytest.log
for SP in 0 1; do
  TNX_SIMT_PLANES=$SP timeout 600 python bench.py --steps 20 --no-cpu-baseline --no-e2e --sustained-s 0 --secondary "" > gpurun_out/r34/bench4_sp$SP.json 2>/dev/null
  TNX_SIMT_PLANES=$SP timeout 600 python bench.py --config cfg5_syc53_m12 --steps 10 --no-cpu-baseline --no-e2e --sustained-s 0 --secondary "" > gpurun_out/r34/bench5_sp$SP.json 2>/dev/null
  TNX_SIMT_PLANES=$SP timeout 600 python bench.py --config cfg3_lattice20 --steps 10 --no-cpu-baseline --no-e2e --sustained-s 0 --secondary "" > gpurun_out/r34/bench3_sp$SP.json 2>/dev/null
  echo "sp$SP"
done
for key in d40 d24; do timeout 300 python tools/prefix_parity.py $key > gpurun_out/r34/pp_$key.json 2>&1; done
