# A/B: staged epilogue through the TMA ring, one tile per pair (old) vs a dedicated double-buffered region with persistent pairs (head)
OUT=gpurun_out
L=paper_2308_03120_b200/libb200mat.so
: > $OUT/ab6.txt
cp abtmp/lib_head.so $L; touch $L
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "memory_input or epilogue or persistent or repeatable" -p no:cacheprovider >> $OUT/ab6.txt 2>&1; echo "pytest head rc=$?" >> $OUT/ab6.txt
BM_GEMM_PERSIST=0 timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -k "memory_input" -p no:cacheprovider >> $OUT/ab6.txt 2>&1; echo "pytest head nopersist rc=$?" >> $OUT/ab6.txt
timeout 300 python tools/epi_bitcheck_8192.py >> $OUT/ab6.txt 2>&1
for round in 1 2 3; do
for v in old head; do
  cp abtmp/lib_$v.so $L; touch $L
  echo "== $v" >> $OUT/ab6.txt
  timeout 300 python tools/epi_mem_probe.py 8192 6 >> $OUT/ab6.txt 2>&1
done
done
cp abtmp/lib_head.so $L
