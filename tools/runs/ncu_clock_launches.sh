mkdir -p gpurun_out/r13
CMD="python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e --no-tf32-probe --sustained-s 0 --profile-out gpurun_out/r13/profile.json"
$CMD > gpurun_out/r13/plain.log 2>&1 && ncu --metrics gpu__time_duration.sum,sm__cycles_elapsed.avg.per_second,sm__cycles_elapsed.max,sm__pipe_tc_cycles_active.avg.pct_of_peak_sustained_active --clock-control none --csv --log-file gpurun_out/r13/launches.csv $CMD > gpurun_out/r13/ncu.log 2>&1; echo "rc=$?"
