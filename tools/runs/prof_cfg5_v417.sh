mkdir -p gpurun_out/r27
python tools/profile_vertex.py cfg5_syc53_m12 417 > gpurun_out/r27/idx.log 2>&1; cat gpurun_out/r27/idx.log | tail -1
I=$(grep -o "gemm launch index [0-9]*" gpurun_out/r27/idx.log | awk '{print $4}')
TNX_DEBUG_PLAN=1 python tools/profile_vertex.py cfg5_syc53_m12 414 > gpurun_out/r27/plan.log 2>&1
ncu --nvtx --nvtx-include "slice/" --set full --clock-control none --import-source on -k regex:gemm_c64 --launch-skip $I -c 1 -o gpurun_out/r27/v417 python tools/profile_vertex.py cfg5_syc53_m12 417 > gpurun_out/r27/ncu.log 2>&1; echo "ncu rc=$?"
