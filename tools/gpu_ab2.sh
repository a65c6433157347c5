# A/B: cluster-scope pipeline barriers (old) vs CTA-scope (head), same box
OUT=gpurun_out
L=paper_2308_03120_b200/libb200mat.so
: > $OUT/ab2.txt
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "gemm or epilogue or memory_input" -p no:cacheprovider >> $OUT/ab2.txt 2>&1; echo "pytest head rc=$?" >> $OUT/ab2.txt
for round in 1 2; do
for v in old head; do
  cp abtmp/lib_$v.so $L; touch $L
  echo "== $v" >> $OUT/ab2.txt
  timeout 120 python tools/gemm32k_sweep.py 8192 10 >> $OUT/ab2.txt 2>&1
  timeout 200 python tools/gemm32k_sweep.py 16384 5 >> $OUT/ab2.txt 2>&1
  timeout 300 python tools/epi_mem_probe.py 8192 6 >> $OUT/ab2.txt 2>&1
done
done
cp abtmp/lib_head.so $L
