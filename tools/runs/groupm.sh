mkdir -p gpurun_out/r46
for G in 8 6 10 12 8; do
  TNX_GEMM_GROUP_M=$G timeout 600 python bench.py --steps 20 --no-cpu-baseline --no-e2e --sustained-s 0 --secondary= > gpurun_out/r46/bench_g$G.json 2>/dev/null
  echo "g$G $(python -c "import json;d=json.loads(open('gpurun_out/r46/bench_g$G.json').read().strip().splitlines()[-1]);print(round(d['value'],1), round(d['clocks']['sm_mhz_cycles']), round(d['roofline']['frac'],3))")"
done
