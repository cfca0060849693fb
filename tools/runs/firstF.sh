mkdir -p gpurun_out/r29
for F in 6 9 12 16; do for v in 417 414; do TNX_GEMM_FIRST=$F python tools/profile_vertex.py cfg5_syc53_m12 $v >> gpurun_out/r29/f$F.log 2>&1; done; done
for F in 6 12; do for key in d40 d24; do TNX_GEMM_FIRST=$F timeout 300 python tools/prefix_parity.py $key > gpurun_out/r29/pp_${key}_f$F.json 2>&1; done; done
