# RZ-bias study: GEMM bias vs promotion interval, then d40/d24 slices vs fixtures
mkdir -p gpurun_out
for P in 1 2 3 6; do
  for K in 0 0.72; do
    TNX_GEMM_PROMOTE=$P TNX_GEMM_FIRST=$P TNX_GEMM_RZC=$K timeout 120 python tools/gemm_bias.py 2048 2048 4096 >> gpurun_out/bias.jsonl 2>>gpurun_out/bias.err
  done
done
TNX_GEMM_RZC=0 timeout 120 python tools/gemm_bias.py 2048 2048 4096 >> gpurun_out/bias.jsonl 2>>gpurun_out/bias.err
TNX_GEMM_RZC=0.72 timeout 120 python tools/gemm_bias.py 2048 2048 4096 >> gpurun_out/bias.jsonl 2>>gpurun_out/bias.err
TNX_GEMM_RZC=0.72 timeout 120 python tools/gemm_bias.py 8192 8192 4096 >> gpurun_out/bias.jsonl 2>>gpurun_out/bias.err
echo bias done
R=cfg4_7x7_d40:27:0-16
R24=cfg4p_7x7_d24:27:0-32
for K in 0 0.72; do
  TNX_GEMM_RZC=$K timeout 300 python tools/prefix_parity.py x --raw $R > gpurun_out/pp_rn_k$K.json 2>&1; echo "d40 k$K rc=$?"
  TNX_GEMM_RZC=$K timeout 300 python tools/prefix_parity.py x --raw $R24 > gpurun_out/pp24_rn_k$K.json 2>&1; echo "d24 k$K rc=$?"
done
TNX_GEMM_RZC=0.72 TNX_GEMM_PROMOTE=2 TNX_GEMM_FIRST=2 timeout 300 python tools/prefix_parity.py x --raw $R > gpurun_out/pp_rn_k0.72_p2.json 2>&1; echo "d40 k.72 p2 rc=$?"
