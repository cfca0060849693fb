mkdir -p gpurun_out/r22
S="8192x16384x512 16384x8192x512 1024x131072x256 2048x16384x512 16384x8192x2048"
python tools/gemm_knobs.py $S > gpurun_out/r22/plain.jsonl 2>&1; echo plain
python tools/gemm_knobs.py --chain=7 $S > gpurun_out/r22/chain.jsonl 2>&1; echo chain
TNX_DEBUG_PLAN=1 python tools/gemm_knobs.py --chain=7 8192x16384x512 > gpurun_out/r22/chain_plan.log 2>&1; echo plan
python tools/run_gemm.py 8192 16384 512 1 1 > /dev/null 2>&1
