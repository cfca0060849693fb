mkdir -p gpurun_out/r26
TNX_BENCH_BACKEND=gloo timeout 900 python bench.py --gpus 8 --steps 3 --warmup 3 --no-cpu-baseline --no-e2e --sustained-s 1 > gpurun_out/r26/bench_8rank_gloo.json 2> gpurun_out/r26/bench_8rank_gloo.err; echo "8rank rc=$?"
timeout 600 python bench.py --force-dist --steps 5 --warmup 3 --no-cpu-baseline --sustained-s 1 > gpurun_out/r26/bench_nccl1.json 2> gpurun_out/r26/bench_nccl1.err; echo "nccl1 rc=$?"
timeout 600 python bench.py --impl reference --gpus 1 --steps 1 --warmup 0 --ref-budget 30 > gpurun_out/r26/ref.json 2> gpurun_out/r26/ref.err; echo "ref rc=$?"
