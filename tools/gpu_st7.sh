# 3xTF32 pair kernel ring: 6 stages (old) vs 7 (head, 225 KB)
OUT=gpurun_out
L=paper_2308_03120_b200/libb200mat.so
: > $OUT/st7.txt
cp abtmp/lib_head.so $L; touch $L
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "gemm_shapes or epilogue_bit or persistent or repeatable" -p no:cacheprovider >> $OUT/st7.txt 2>&1; echo "pytest st7 rc=$?" >> $OUT/st7.txt
for round in 1 2; do
for v in old head; do
  cp abtmp/lib_$v.so $L; touch $L
  echo "== $v" >> $OUT/st7.txt
  for n in 8192 16384; do timeout 200 python tools/gemm32k_sweep.py $n 10 >> $OUT/st7.txt 2>&1; done
done
done
for v in old head; do
  cp abtmp/lib_$v.so $L; touch $L
  echo "== $v 32k" >> $OUT/st7.txt
  timeout 300 python tools/gemm32k_sweep.py 32768 3 >> $OUT/st7.txt 2>&1
done
cp abtmp/lib_old.so $L
