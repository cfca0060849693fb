mkdir -p gpurun_out/r38
CMD="python bench.py --steps 1 --warmup 0 --no-cpu-baseline --no-e2e --no-tf32-probe --sustained-s 0 --secondary= --profile-out gpurun_out/r38/profile.json"
$CMD > gpurun_out/r38/plain.log 2>&1 && ncu --metrics gpu__time_duration.sum,sm__cycles_elapsed.max,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/r38/launches.csv $CMD > gpurun_out/r38/ncu.log 2>&1; echo "rc=$?"
