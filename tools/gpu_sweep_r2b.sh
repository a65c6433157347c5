# after the barrier-scope fix: K-pass / raster-group / persistence sweep
OUT=gpurun_out
: > $OUT/sweep_r2b.txt
nvidia-smi --query-gpu=clocks.sm,power.draw,clocks_event_reasons.active --format=csv,noheader -lms 200 > $OUT/sweep_r2b_clk.csv &
SMI=$!
for kp in 8192 16384 0; do
  for g in 4 8; do
    BM_GEMM_KPASS=$kp BM_GEMM_GROUP=$g timeout 300 python tools/gemm32k_sweep.py 32768 3 >> $OUT/sweep_r2b.txt 2>&1
  done
done
for p in 0 1 0 1; do
  for n in 8192 16384; do
    echo "persist=$p" >> $OUT/sweep_r2b.txt
    BM_GEMM_PERSIST=$p timeout 200 python tools/gemm32k_sweep.py $n 10 >> $OUT/sweep_r2b.txt 2>&1
  done
done
kill $SMI
timeout 300 python tools/fusion_probe.py 8192 f32 >> $OUT/sweep_r2b.txt 2>&1
timeout 300 python tools/epi_mem_probe.py 8192 8 >> $OUT/sweep_r2b.txt 2>&1
