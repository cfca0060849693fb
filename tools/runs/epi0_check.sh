mkdir -p gpurun_out/r20
timeout 600 python -m pytest tests/test_gpu_parity.py -q -m gpu -x -k "gemm or golden or circuit" > gpurun_out/r20/pytest.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/r20/pytest.log
S="8192x16384x512 32768x4096x512 16384x8192x2048 4096x32768x1024 1024x131072x256"
python tools/gemm_knobs.py $S > gpurun_out/r20/knobs.jsonl 2>&1; echo knobs
TNX_GEMM_DEBUG=1 python tools/gemm_knobs.py $S > gpurun_out/r20/notma.jsonl 2>&1; echo notma
timeout 600 python bench.py --steps 20 --no-cpu-baseline --no-e2e --sustained-s 0 > gpurun_out/r20/bench.json 2> gpurun_out/r20/bench.err; echo bench
timeout 600 python bench.py --config cfg5_syc53_m12 --steps 10 --no-cpu-baseline --no-e2e --sustained-s 0 > gpurun_out/r20/bench5.json 2> gpurun_out/r20/bench5.err; echo bench5
timeout 600 python bench.py --config cfg2_5reg100 --steps 10 --no-cpu-baseline --no-e2e --sustained-s 0 > gpurun_out/r20/bench2.json 2> gpurun_out/r20/bench2.err; echo bench2
