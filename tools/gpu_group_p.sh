# raster group sweep with persistent pairs (default)
OUT=gpurun_out
: > $OUT/group_p.txt
for round in 1 2; do
for g in 2 4 8 16; do
  for n in 8192 16384; do
    BM_GEMM_GROUP=$g timeout 200 python tools/gemm32k_sweep.py $n 10 >> $OUT/group_p.txt 2>&1
  done
done
done
