mkdir -p gpurun_out/r23
timeout 1000 python tools/fuzz_gpu.py 900 5000 > gpurun_out/r23/fuzz.log 2>&1; echo "fuzz rc=$?"; tail -2 gpurun_out/r23/fuzz.log
CMD="python bench.py --steps 1 --warmup 0 --no-cpu-baseline --no-e2e --no-tf32-probe --sustained-s 0 --profile-out gpurun_out/r23/profile.json"
$CMD > gpurun_out/r23/plain.log 2>&1 && ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,sm__cycles_elapsed.max --clock-control none --csv --log-file gpurun_out/r23/launches_dram.csv $CMD > gpurun_out/r23/ncu.log 2>&1; echo "launch dram rc=$?"
