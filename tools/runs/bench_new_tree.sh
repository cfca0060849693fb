mkdir -p gpurun_out/r7
timeout 900 python bench.py --profile-out gpurun_out/r7/profile.json > gpurun_out/r7/bench_default.json 2> gpurun_out/r7/bench_default.err; echo "bench rc=$?"
timeout 300 python tools/prefix_parity.py x --raw cfg4_7x7_d40:27:0-16 > gpurun_out/r7/d40.json 2>&1; echo "d40 rc=$?"
for ws in 30; do timeout 600 python bench.py --ws $ws --steps 5 --no-cpu-baseline --no-e2e --sustained-s 0 > gpurun_out/r7/bench_ws$ws.json 2>gpurun_out/r7/bench_ws$ws.err; echo "ws$ws rc=$?"; done
