mkdir -p gpurun_out/r42
for c in cfg1_3reg50 cfg2_5reg100 cfg3_lattice20 cfg3g_lattice20 cfg4g_7x7_d40 cfg4d_7x7_d40_diag cfg5_syc53_m12; do
  timeout 600 python bench.py --config $c --steps 5 --no-cpu-baseline --no-e2e --sustained-s 0 --secondary= > gpurun_out/r42/bench_$c.json 2> gpurun_out/r42/bench_$c.err; echo "$c rc=$?"
done
timeout 600 python bench.py --ws 30 --steps 3 --no-cpu-baseline --no-e2e --sustained-s 0 --secondary= > gpurun_out/r42/bench_cfg4_ws30.json 2> gpurun_out/r42/bench_cfg4_ws30.err; echo "ws30 rc=$?"
timeout 600 python bench.py --config cfg5_syc53_m12 --ws 30 --steps 2 --no-cpu-baseline --no-e2e --sustained-s 0 --secondary= > gpurun_out/r42/bench_cfg5_ws30.json 2> gpurun_out/r42/bench_cfg5_ws30.err; echo "cfg5 ws30 rc=$?"
timeout 2200 python tools/fuzz_gpu.py 2100 20000 > gpurun_out/r42/fuzz.log 2>&1; echo "fuzz rc=$?"; tail -1 gpurun_out/r42/fuzz.log
