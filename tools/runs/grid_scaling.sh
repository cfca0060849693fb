mkdir -p gpurun_out/r45
S="16384x8192x2048"
for NP in 74 56 37 18; do
  TNX_GEMM_MAXPAIRS=$NP TNX_GEMM_DEBUG=34 python tools/gemm_knobs.py $S > gpurun_out/r45/tma_np$NP.jsonl 2>&1
  TNX_GEMM_MAXPAIRS=$NP python tools/gemm_knobs.py $S > gpurun_out/r45/full_np$NP.jsonl 2>&1
  echo np$NP
done
