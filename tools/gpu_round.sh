#!/bin/bash
# One GPU evidence session: full GPU test suite, smoke(), default bench,
# reference arm, 2-rank gloo bench on the shared GPU, MMA/FFMA ceilings, ncu
# launch list of the bench command, ncu full captures of the dominant GEMM
# shape (16384 x 8192 x 2048 in the min-fill cfg4 workload), the permute and
# the SIMT kernels.  Summarise with tools/summarize_profiles.py.
set -u
O=gpurun_out
mkdir -p $O
timeout 1200 python -m pytest tests -q -m gpu > $O/pytest_gpu.log 2>&1; echo "pytest_gpu rc=$?"; tail -3 $O/pytest_gpu.log
timeout 300 python __graft_entry__.py > $O/smoke.log 2>&1; echo "smoke rc=$?"; tail -2 $O/smoke.log
timeout 900 python bench.py > $O/bench_default.log 2>$O/bench_default.err; echo "bench rc=$?"
timeout 600 python bench.py --impl reference --steps 2 --warmup 0 --ref-budget 45 > $O/bench_reference.log 2>$O/bench_reference.err; echo "ref rc=$?"
TNX_BENCH_BACKEND=gloo timeout 600 python bench.py --gpus 2 --steps 4 --warmup 3 --no-cpu-baseline --sustained-s 2 > $O/bench_2rank_gloo.log 2>$O/bench_2rank_gloo.err; echo "2rank rc=$?"
timeout 300 python tools/mma_peak.py --sustained-s 5 --out $O/mma_peak.json > $O/mma_peak.log 2>&1; echo "peak rc=$?"
CMD="python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e --no-tf32-probe --sustained-s 0 --secondary="
$CMD > $O/plain_launch.log 2>&1 && ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches.csv $CMD > $O/ncu_launch.log 2>&1; echo "ncu launches rc=$?"
CMD2="python bench.py --steps 1 --warmup 0 --no-cpu-baseline --no-e2e --no-tf32-probe --sustained-s 0 --secondary= --profile-out $O/profile.json"
$CMD2 > $O/plain_launch2.log 2>&1 && ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,sm__cycles_elapsed.max --clock-control none --csv --log-file $O/launches_dram.csv $CMD2 > $O/ncu_launch2.log 2>&1; echo "ncu launches dram rc=$?"
python tools/run_gemm.py 16384 8192 2048 1 2 > $O/plain_gemm.log 2>&1 && ncu --set full --clock-control none --import-source on -k regex:gemm_c64 -c 1 -o $O/prof_gemm_full python tools/run_gemm.py 16384 8192 2048 1 1 > $O/ncu_gemm.log 2>&1; echo "ncu gemm rc=$?"
python tools/run_perm.py 3 > $O/plain_perm.log 2>&1 && ncu --set full --clock-control none --import-source on -k regex:"perm|gather" -c 2 -o $O/prof_perm_full python tools/run_perm.py 1 > $O/ncu_perm.log 2>&1; echo "ncu perm rc=$?"
python tools/run_simt.py 3 > $O/plain_simt.log 2>&1 && ncu --set full --clock-control none --import-source on -k regex:"simt" -c 2 -o $O/prof_simt_full python tools/run_simt.py 1 > $O/ncu_simt.log 2>&1; echo "ncu simt rc=$?"
