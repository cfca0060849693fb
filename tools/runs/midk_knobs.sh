mkdir -p gpurun_out/r18
S="8192x16384x512 32768x4096x512 16384x8192x512 16384x8192x2048 4096x32768x1024"
python tools/gemm_knobs.py $S > gpurun_out/r18/default.jsonl 2>&1; echo default
TNX_GEMM_FIRST=12 python tools/gemm_knobs.py $S > gpurun_out/r18/first12.jsonl 2>&1; echo first12
TNX_GEMM_FIRST=32 TNX_GEMM_PROMOTE=32 python tools/gemm_knobs.py $S > gpurun_out/r18/p32.jsonl 2>&1; echo p32
TNX_GEMM_PROMOTE=4 TNX_GEMM_FIRST=8 python tools/gemm_knobs.py $S > gpurun_out/r18/p4.jsonl 2>&1; echo p4
TNX_GEMM_DEBUG=1 python tools/gemm_knobs.py $S > gpurun_out/r18/notma.jsonl 2>&1; echo notma
TNX_GEMM_GROUP_M=4 python tools/gemm_knobs.py $S > gpurun_out/r18/g4.jsonl 2>&1; echo g4
TNX_GEMM_GROUP_M=16 python tools/gemm_knobs.py $S > gpurun_out/r18/g16.jsonl 2>&1; echo g16
python tools/run_gemm.py 8192 16384 512 1 2 > /dev/null 2>&1; ncu --set full --clock-control none --import-source on -k regex:gemm_c64 -c 1 -o gpurun_out/r18/midk python tools/run_gemm.py 8192 16384 512 1 1 > gpurun_out/r18/ncu.log 2>&1; echo ncu
