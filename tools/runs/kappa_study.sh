# kappa x promotion sweep: random-GEMM bias + d40 (greedy tree) and d24 slices
mkdir -p gpurun_out/kappa
R=cfg4g_7x7_d40:27:0-16
R24=cfg4p_7x7_d24:27:0-32
for PF in "3 6" "2 2" "3 3"; do
  set -- $PF
  for K in 0.3 0.45 0.6; do
    tag=p$1f$2_k$K
    TNX_GEMM_PROMOTE=$1 TNX_GEMM_FIRST=$2 TNX_GEMM_RZC=$K timeout 120 python tools/gemm_bias.py 2048 2048 4096 > gpurun_out/kappa/bias_$tag.json 2>&1
    TNX_GEMM_PROMOTE=$1 TNX_GEMM_FIRST=$2 TNX_GEMM_RZC=$K timeout 300 python tools/prefix_parity.py x --raw $R > gpurun_out/kappa/d40_$tag.json 2>&1
    TNX_GEMM_PROMOTE=$1 TNX_GEMM_FIRST=$2 TNX_GEMM_RZC=$K timeout 300 python tools/prefix_parity.py x --raw $R24 > gpurun_out/kappa/d24_$tag.json 2>&1
    echo "$tag done"
  done
done
for PF in "3 6" "2 2" "3 3"; do
  set -- $PF
  TNX_GEMM_PROMOTE=$1 TNX_GEMM_FIRST=$2 timeout 300 python bench.py --config cfg4g_7x7_d40 --steps 20 --warmup 3 --no-cpu-baseline --no-e2e --sustained-s 0 > gpurun_out/kappa/bench_p$1f$2.json 2> gpurun_out/kappa/bench_p$1f$2.err
  echo "bench p$1f$2 rc=$?"
done
