mkdir -p gpurun_out/r6
timeout 300 python tools/prefix_parity.py x --raw cfg4g_7x7_d40:27:0-16 > gpurun_out/r6/d40.json 2>&1; echo "d40 rc=$?"
timeout 300 python tools/prefix_parity.py x --raw cfg4p_7x7_d24:27:0-32 > gpurun_out/r6/d24.json 2>&1; echo "d24 rc=$?"
TNX_BENCH_BACKEND=gloo timeout 600 python bench.py --gpus 2 --steps 4 --warmup 3 --no-cpu-baseline --sustained-s 2 > gpurun_out/r6/bench_2rank.json 2> gpurun_out/r6/bench_2rank.err; echo "2rank rc=$?"
timeout 900 python bench.py --config cfg4g_7x7_d40 > gpurun_out/r6/bench_default.json 2> gpurun_out/r6/bench_default.err; echo "bench rc=$?"
tail -c 1500 gpurun_out/r6/bench_default.json
