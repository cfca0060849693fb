mkdir -p gpurun_out/r24
for PF in "3 6" "4 8" "5 10" "6 12"; do
  set -- $PF
  for key in d40 d24 d40g; do
    TNX_GEMM_PROMOTE=$1 TNX_GEMM_FIRST=$2 timeout 300 python tools/prefix_parity.py $key > gpurun_out/r24/pp_${key}_p$1.json 2>&1
  done
  TNX_GEMM_PROMOTE=$1 TNX_GEMM_FIRST=$2 timeout 300 python tools/gemm_bias.py 2048 2048 4096 > gpurun_out/r24/bias_p$1.json 2>&1
  TNX_GEMM_PROMOTE=$1 TNX_GEMM_FIRST=$2 timeout 600 python bench.py --steps 20 --no-cpu-baseline --no-e2e --sustained-s 6 > gpurun_out/r24/bench_p$1.json 2> gpurun_out/r24/bench_p$1.err
  echo "p$1 done"
done
