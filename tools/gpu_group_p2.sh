# raster group 4 vs 8 by size, interleaved
OUT=gpurun_out
: > $OUT/group_p2.txt
for round in 1 2 3; do
for n in 4096 6144 8192 12288; do
  for g in 4 8; do
    BM_GEMM_GROUP=$g timeout 200 python tools/gemm32k_sweep.py $n 10 >> $OUT/group_p2.txt 2>&1
  done
done
done
