nvidia-smi --query-gpu=index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active --format=csv -lms 200 > gpurun_out/clocks_sweep32k.csv &
SMI=$!
for g in 2 4 8 16; do for kp in 4096 8192 16384; do
  BM_GEMM_GROUP=$g BM_GEMM_KPASS=$kp timeout 120 python tools/gemm32k_sweep.py 32768 3 >> gpurun_out/sweep32k.txt 2>&1
done; done
kill $SMI
