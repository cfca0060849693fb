mkdir -p gpurun_out/r28
for v in 417 414 418; do python tools/profile_vertex.py cfg5_syc53_m12 $v >> gpurun_out/r28/base.log 2>&1; done
for v in 417 414; do TNX_GEMM_DEBUG=2 python tools/profile_vertex.py cfg5_syc53_m12 $v >> gpurun_out/r28/nostore.log 2>&1; done
for S in 2 4 6; do for v in 417 414; do TNX_GEMM_STAGGER=$S python tools/profile_vertex.py cfg5_syc53_m12 $v >> gpurun_out/r28/stagger$S.log 2>&1; done; done
for S in 0 4; do TNX_GEMM_STAGGER=$S timeout 600 python bench.py --config cfg5_syc53_m12 --steps 10 --no-cpu-baseline --no-e2e --sustained-s 0 > gpurun_out/r28/bench5_s$S.json 2>/dev/null; TNX_GEMM_STAGGER=$S timeout 600 python bench.py --steps 20 --no-cpu-baseline --no-e2e --sustained-s 0 > gpurun_out/r28/bench4_s$S.json 2>/dev/null; echo "s$S"; done
