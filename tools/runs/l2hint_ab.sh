mkdir -p gpurun_out/r15
for H in 0 1; do
  TNX_GEMM_L2HINT=$H python tools/run_gemm.py 16384 8192 2048 1 3 > gpurun_out/r15/plain_h$H.log 2>&1
  TNX_GEMM_L2HINT=$H ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_bytes.sum,sm__cycles_elapsed.max,sm__cycles_elapsed.avg.per_second --clock-control none -k regex:gemm_c64 -c 1 --csv python tools/run_gemm.py 16384 8192 2048 1 1 > gpurun_out/r15/ncu_h$H.csv 2>&1
  TNX_GEMM_L2HINT=$H ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_bytes.sum,sm__cycles_elapsed.max --clock-control none -k regex:gemm_c64 -c 1 --csv python tools/run_gemm.py 8192 8192 4096 1 1 > gpurun_out/r15/ncu8k_h$H.csv 2>&1
  TNX_GEMM_L2HINT=$H timeout 600 python bench.py --steps 20 --no-cpu-baseline --no-e2e --sustained-s 10 > gpurun_out/r15/bench_h$H.json 2> gpurun_out/r15/bench_h$H.err
  echo "h$H done"
done
