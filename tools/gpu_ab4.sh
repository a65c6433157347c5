# A/B: staged epilogue kernels with (old) and without (head) the direct-load fallback path compiled in
OUT=gpurun_out
L=paper_2308_03120_b200/libb200mat.so
: > $OUT/ab4.txt
for round in 1 2 3; do
for v in old head; do
  cp abtmp/lib_$v.so $L; touch $L
  echo "== $v" >> $OUT/ab4.txt
  timeout 300 python tools/epi_mem_probe.py 8192 8 >> $OUT/ab4.txt 2>&1
done
done
cp abtmp/lib_head.so $L
