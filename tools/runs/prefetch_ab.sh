mkdir -p gpurun_out/r19
S="8192x16384x512 32768x4096x512 16384x8192x2048 4096x32768x1024 1024x131072x256"
for PF in 0 2 4 8; do TNX_GEMM_PREFETCH=$PF python tools/gemm_knobs.py $S > gpurun_out/r19/pf$PF.jsonl 2>&1; echo pf$PF; done
for PF in 0 4; do TNX_GEMM_PREFETCH=$PF timeout 600 python bench.py --steps 20 --no-cpu-baseline --no-e2e --sustained-s 0 > gpurun_out/r19/bench_pf$PF.json 2> gpurun_out/r19/bench_pf$PF.err; echo bench$PF; done
for PF in 0 4; do TNX_GEMM_PREFETCH=$PF timeout 600 python bench.py --config cfg5_syc53_m12 --steps 10 --no-cpu-baseline --no-e2e --sustained-s 0 > gpurun_out/r19/bench5_pf$PF.json 2> gpurun_out/r19/bench5_pf$PF.err; echo bench5_$PF; done
