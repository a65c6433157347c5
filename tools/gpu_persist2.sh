# persistent pair GEMM: sustained A/B (50 reps, clocks logged) and the fusion probe in both orders
OUT=gpurun_out
: > $OUT/persist2.txt
for p in 1 0 1 0; do
  echo "== persist=$p fusion" >> $OUT/persist2.txt
  BM_GEMM_PERSIST=$p timeout 300 python tools/fusion_probe.py 8192 f32 >> $OUT/persist2.txt 2>&1
done
for p in 1 0 1 0; do
  echo "== persist=$p 8192 x50" >> $OUT/persist2.txt
  nvidia-smi --query-gpu=clocks.sm,power.draw,temperature.gpu --format=csv,noheader -lms 200 > $OUT/clk_$p.csv &
  SMI=$!
  BM_GEMM_PERSIST=$p timeout 200 python tools/gemm32k_sweep.py 8192 50 >> $OUT/persist2.txt 2>&1
  kill $SMI
  sort -t, -k1 -n $OUT/clk_$p.csv | awk -F, '{a[NR]=$1} END {print "median sm clock", a[int(NR/2)]}' >> $OUT/persist2.txt
  tail -3 $OUT/clk_$p.csv >> $OUT/persist2.txt
done
