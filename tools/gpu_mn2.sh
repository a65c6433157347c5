# MN-major operands (3-D maps) vs K-major copies, same binary, BM_GEMM_MN=1 / 0
OUT=gpurun_out
: > $OUT/mn2.txt
BM_GEMM_MN=1 timeout 1200 python -m pytest tests/test_gpu_parity.py -x -q -k "gemm or epilogue or memory_input or persistent or repeatable or random_programs" -p no:cacheprovider >> $OUT/mn2.txt 2>&1; echo "pytest MN=1 rc=$?" >> $OUT/mn2.txt
for round in 1 2; do
for v in 0 1; do
  echo "== MN=$v" >> $OUT/mn2.txt
  for n in 8192 16384; do BM_GEMM_MN=$v timeout 200 python tools/gemm32k_sweep.py $n 10 >> $OUT/mn2.txt 2>&1; done
done
done
