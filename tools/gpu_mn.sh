# MN-major operands read in place (head) vs K-major hi/lo copies (old)
OUT=gpurun_out
L=paper_2308_03120_b200/libb200mat.so
: > $OUT/mn.txt
cp abtmp/lib_head.so $L; touch $L
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_baseline_shapes.py tests/test_gpu_reference_suite.py -x -q -k "gemm or epilogue or memory_input or persistent or repeatable or random_programs or operand or matmul or linalg" -p no:cacheprovider >> $OUT/mn.txt 2>&1; echo "pytest head rc=$?" >> $OUT/mn.txt
BM_GEMM_MN=0 timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -k "gemm_shapes or epilogue_bit or repeatable" -p no:cacheprovider >> $OUT/mn.txt 2>&1; echo "pytest head MN=0 rc=$?" >> $OUT/mn.txt
for round in 1 2; do
for v in old head; do
  cp abtmp/lib_$v.so $L; touch $L
  echo "== $v" >> $OUT/mn.txt
  for n in 8192 16384; do timeout 200 python tools/gemm32k_sweep.py $n 10 >> $OUT/mn.txt 2>&1; done
done
done
cp abtmp/lib_head.so $L
