mkdir -p gpurun_out/r10
timeout 900 python -m pytest tests/test_gpu_configs.py tests/test_gpu_northstar.py -m gpu -q -s -k "not d40-key and not d40r-key" > gpurun_out/r10/pytest.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/r10/pytest.log
timeout 900 python bench.py > gpurun_out/r10/bench_default.json 2> gpurun_out/r10/bench_default.err; echo "bench rc=$?"
timeout 600 python bench.py --impl reference --steps 2 --warmup 1 --ref-budget 45 > gpurun_out/r10/bench_ref.json 2> gpurun_out/r10/bench_ref.err; echo "ref rc=$?"
TNX_BENCH_BACKEND=gloo timeout 600 python bench.py --gpus 2 --steps 4 --warmup 3 --no-cpu-baseline --sustained-s 2 > gpurun_out/r10/bench_2rank.json 2> gpurun_out/r10/bench_2rank.err; echo "2rank rc=$?"
