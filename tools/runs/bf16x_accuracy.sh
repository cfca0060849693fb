mkdir -p gpurun_out/r11
for K in 0 0.35 0.5; do
  PREC=2 TNX_GEMM_RZC=$K timeout 120 python tools/gemm_bias.py 2048 2048 4096 >> gpurun_out/r11/bias.jsonl 2>&1
  PREC=1 TNX_GEMM_RZC=$K timeout 120 python tools/gemm_bias.py 2048 2048 4096 >> gpurun_out/r11/bias.jsonl 2>&1
  TNX_GEMM_RZC=$K timeout 300 python tools/prefix_parity.py x --raw cfg4g_7x7_d40:27:0-16 --precision tf32-bf16x > gpurun_out/r11/d40g_k$K.json 2>&1
  TNX_GEMM_RZC=$K timeout 300 python tools/prefix_parity.py x --raw cfg4p_7x7_d24:27:0-32 --precision tf32-bf16x > gpurun_out/r11/d24_k$K.json 2>&1
  echo "k$K done"
done
timeout 300 python bench.py --precision tf32-bf16x --steps 20 --no-cpu-baseline --no-e2e --sustained-s 0 > gpurun_out/r11/bench_bf16x.json 2> gpurun_out/r11/bench_bf16x.err; echo "bench rc=$?"
