mkdir -p gpurun_out/r25
for K in 0.25 0.35 0.45; do
  for key in d40 d40r d24 d40g; do
    TNX_GEMM_RZC=$K timeout 300 python tools/prefix_parity.py $key > gpurun_out/r25/pp_${key}_k$K.json 2>&1
  done
  echo "k$K done"
done
for key in d40 d40r; do TNX_PRECISION=fp32 timeout 600 python tools/prefix_parity.py $key --precision fp32 > gpurun_out/r25/pp_${key}_fp32.json 2>&1; done
echo fp32 done
