mkdir -p gpurun_out/r40
for DBG in 0 16 2; do for v in 1456 1467 1475 1473 1477; do TNX_GEMM_DEBUG=$DBG python tools/profile_vertex.py cfg4_7x7_d40 $v >> gpurun_out/r40/dbg$DBG.log 2>&1; done; done
for DBG in 0 16; do for v in 417 414; do TNX_GEMM_DEBUG=$DBG python tools/profile_vertex.py cfg5_syc53_m12 $v >> gpurun_out/r40/c5dbg$DBG.log 2>&1; done; done
