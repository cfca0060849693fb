mkdir -p gpurun_out/r43
S="16384x8192x2048 8192x16384x512 4096x32768x1024"
for DBG in 0 32 34 2 1; do TNX_GEMM_DEBUG=$DBG python tools/gemm_knobs.py $S > gpurun_out/r43/dbg$DBG.jsonl 2>&1; echo "dbg$DBG"; done
python tools/run_gemm.py 16384 8192 2048 1 1 > /dev/null 2>&1
TNX_GEMM_DEBUG=34 ncu --metrics gpu__time_duration.sum,sm__cycles_elapsed.max,lts__throughput.avg.pct_of_peak_sustained_elapsed,l1tex__m_xbar2l1tex_read_bytes.sum,dram__bytes_read.sum --clock-control none -k regex:gemm_c64 -c 1 --csv python tools/run_gemm.py 16384 8192 2048 1 1 > gpurun_out/r43/ncu_tma_only.csv 2>&1
ncu --metrics gpu__time_duration.sum,sm__cycles_elapsed.max,lts__throughput.avg.pct_of_peak_sustained_elapsed,l1tex__m_xbar2l1tex_read_bytes.sum,dram__bytes_read.sum --clock-control none -k regex:gemm_c64 -c 1 --csv python tools/run_gemm.py 16384 8192 2048 1 1 > gpurun_out/r43/ncu_full.csv 2>&1
echo done
