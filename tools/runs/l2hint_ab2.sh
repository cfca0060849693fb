mkdir -p gpurun_out/r16
for rep in 1 2; do
for H in 0 1 2 3; do
  TNX_GEMM_L2HINT=$H timeout 600 python bench.py --steps 20 --no-cpu-baseline --no-e2e --sustained-s 6 > gpurun_out/r16/bench_h${H}_$rep.json 2> gpurun_out/r16/bench_h${H}_$rep.err
  echo "h$H rep$rep done"
done
done
for shp in "8192 16384 512" "32768 4096 512"; do
  set -- $shp
  ncu --metrics gpu__time_duration.sum,sm__cycles_elapsed.max,sm__pipe_tc_cycles_active.avg.pct_of_peak_sustained_active,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:gemm_c64 -c 1 --csv python tools/run_gemm.py $1 $2 $3 1 1 > gpurun_out/r16/ncu_$1_$2_$3.csv 2>&1
done
