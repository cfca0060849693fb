mkdir -p gpurun_out/r12
python tools/run_gemm.py 16384 8192 2048 1 3 > gpurun_out/r12/plain_a.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:gemm_c64 -c 1 -o gpurun_out/r12/gemm_16k_8k_2k python tools/run_gemm.py 16384 8192 2048 1 1 > gpurun_out/r12/ncu_a.log 2>&1; echo "a rc=$?"
python tools/run_gemm.py 4096 32768 1024 1 3 > gpurun_out/r12/plain_b.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:gemm_c64 -c 1 -o gpurun_out/r12/gemm_4k_32k_1k python tools/run_gemm.py 4096 32768 1024 1 1 > gpurun_out/r12/ncu_b.log 2>&1; echo "b rc=$?"
CMD="python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e --no-tf32-probe --sustained-s 0"
$CMD > gpurun_out/r12/plain_launch.log 2>&1 && ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/r12/launches.csv $CMD > gpurun_out/r12/ncu_launch.log 2>&1; echo "launches rc=$?"
