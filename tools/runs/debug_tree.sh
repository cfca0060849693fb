mkdir -p gpurun_out/r8
timeout 600 python tools/parity_slice.py cfg4_7x7_d40 0 27 > gpurun_out/r8/ps_tc.log 2>&1; echo "tc rc=$?"
TNX_PRECISION=fp32 timeout 900 python tools/parity_slice.py cfg4_7x7_d40 0 27 > gpurun_out/r8/ps_fp32.log 2>&1; echo "fp32 rc=$?"
timeout 300 python tools/prefix_parity.py x --raw cfg4_7x7_d40:27:0-4 --direct 0 > gpurun_out/r8/nodirect.json 2>&1; echo "nodirect rc=$?"
TNX_PRECISION=fp32 timeout 300 python tools/prefix_parity.py x --raw cfg4_7x7_d40:27:0-4 --precision fp32 > gpurun_out/r8/fp32.json 2>&1; echo "fp32 raw rc=$?"
