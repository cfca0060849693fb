mkdir -p gpurun_out
timeout 300 python tools/mma_peak.py --sustained-s 5 --out gpurun_out/mma_peak.json > gpurun_out/mma_peak.log 2>&1; echo "peak rc=$?"; tail -2 gpurun_out/mma_peak.log
R=cfg4_7x7_d40:27:0-16
timeout 300 python tools/prefix_parity.py x --raw $R > gpurun_out/pp_default.json 2>&1; echo "default rc=$?"
TNX_GEMM_FIRST=3 timeout 300 python tools/prefix_parity.py x --raw $R > gpurun_out/pp_p3f3.json 2>&1; echo "p3f3 rc=$?"
TNX_GEMM_PROMOTE=2 TNX_GEMM_FIRST=2 timeout 300 python tools/prefix_parity.py x --raw $R > gpurun_out/pp_p2.json 2>&1; echo "p2 rc=$?"
TNX_GEMM_PROMOTE=1 TNX_GEMM_FIRST=1 timeout 300 python tools/prefix_parity.py x --raw $R > gpurun_out/pp_p1.json 2>&1; echo "p1 rc=$?"
timeout 600 python tools/prefix_parity.py x --raw $R --precision fp32 > gpurun_out/pp_fp32.json 2>&1; echo "fp32 rc=$?"
timeout 300 python tools/prefix_parity.py x --raw $R --direct 0 > gpurun_out/pp_nodirect.json 2>&1; echo "nodirect rc=$?"
R24=cfg4p_7x7_d24:27:0-32
timeout 300 python tools/prefix_parity.py x --raw $R24 > gpurun_out/pp24_default.json 2>&1; echo "d24 default rc=$?"
TNX_GEMM_PROMOTE=1 TNX_GEMM_FIRST=1 timeout 300 python tools/prefix_parity.py x --raw $R24 > gpurun_out/pp24_p1.json 2>&1; echo "d24 p1 rc=$?"
timeout 600 python tools/prefix_parity.py x --raw $R24 --precision fp32 > gpurun_out/pp24_fp32.json 2>&1; echo "d24 fp32 rc=$?"
