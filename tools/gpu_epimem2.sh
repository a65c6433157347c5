OUT=gpurun_out
: > $OUT/epimem2.txt
for g in 4 2 1 8; do
for p in 0 1; do
  echo "== group=$g persist=$p" >> $OUT/epimem2.txt
  BM_GEMM_EPI_GROUP=$g BM_GEMM_PERSIST=$p timeout 300 python tools/epi_mem_probe.py 8192 8 >> $OUT/epimem2.txt 2>&1
done
done
