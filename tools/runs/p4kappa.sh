mkdir -p gpurun_out/r35
for K in 0.28 0.32 0.36; do
  for key in d40 d40r d24 d40g; do
    TNX_GEMM_PROMOTE=4 TNX_GEMM_FIRST=8 TNX_GEMM_RZC=$K timeout 300 python tools/prefix_parity.py $key > gpurun_out/r35/pp_${key}_k$K.json 2>&1
  done
  echo "k$K"
done
for key in d40 d40r d24 d40g; do TNX_GEMM_PROMOTE=4 TNX_GEMM_FIRST=6 TNX_GEMM_RZC=0.32 timeout 300 python tools/prefix_parity.py $key > gpurun_out/r35/pp_${key}_f6.json 2>&1; done
