mkdir -p gpurun_out/r14
timeout 900 python bench.py > gpurun_out/r14/bench_default.json 2> gpurun_out/r14/bench_default.err; echo "bench rc=$?"
for c in cfg1_3reg50 cfg3_lattice20 cfg3g_lattice20 cfg2_5reg100 cfg5_syc53_m12 cfg4g_7x7_d40; do
  timeout 600 python bench.py --config $c --steps 5 --no-cpu-baseline --no-e2e --sustained-s 0 > gpurun_out/r14/bench_$c.json 2> gpurun_out/r14/bench_$c.err; echo "$c rc=$?"
done
timeout 600 python bench.py --config cfg4_7x7_d40 --ws 30 --steps 3 --no-cpu-baseline --no-e2e --sustained-s 0 > gpurun_out/r14/bench_cfg4_ws30.json 2> gpurun_out/r14/bench_cfg4_ws30.err; echo "ws30 rc=$?"
