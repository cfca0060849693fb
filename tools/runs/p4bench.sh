mkdir -p gpurun_out/r36
for rep in 1 2; do
  timeout 600 python bench.py --steps 20 --no-cpu-baseline --no-e2e --sustained-s 6 --secondary= > gpurun_out/r36/bench_p3_$rep.json 2>/dev/null
  TNX_GEMM_PROMOTE=4 TNX_GEMM_FIRST=6 TNX_GEMM_RZC=0.32 timeout 600 python bench.py --steps 20 --no-cpu-baseline --no-e2e --sustained-s 6 --secondary= > gpurun_out/r36/bench_p4_$rep.json 2>/dev/null
done
for c in cfg5_syc53_m12 cfg2_5reg100; do
  timeout 600 python bench.py --config $c --steps 10 --no-cpu-baseline --no-e2e --sustained-s 0 --secondary= > gpurun_out/r36/b_${c}_p3.json 2>/dev/null
  TNX_GEMM_PROMOTE=4 TNX_GEMM_FIRST=6 TNX_GEMM_RZC=0.32 timeout 600 python bench.py --config $c --steps 10 --no-cpu-baseline --no-e2e --sustained-s 0 --secondary= > gpurun_out/r36/b_${c}_p4.json 2>/dev/null
done
TNX_GEMM_PROMOTE=4 TNX_GEMM_FIRST=6 TNX_GEMM_RZC=0.32 python tools/gemm_bias.py 2048 2048 4096 > gpurun_out/r36/bias_p4.json 2>&1
python tools/gemm_bias.py 2048 2048 4096 > gpurun_out/r36/bias_p3.json 2>&1
