# persistent pair GEMM with dynamic tile claiming: parity, then A/B against one pair per tile
OUT=gpurun_out
: > $OUT/persist.txt
BM_GEMM_PERSIST=1 timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "gemm or epilogue" -p no:cacheprovider >> $OUT/persist.txt 2>&1; echo "pytest persist rc=$?" >> $OUT/persist.txt
for round in 1 2; do
for p in 0 1; do
  for n in 8192 16384; do
    echo "== persist=$p" >> $OUT/persist.txt
    BM_GEMM_PERSIST=$p timeout 200 python tools/gemm32k_sweep.py $n 10 >> $OUT/persist.txt 2>&1
  done
done
done
for p in 0 1; do
  echo "== persist=$p 32k" >> $OUT/persist.txt
  BM_GEMM_PERSIST=$p timeout 300 python tools/gemm32k_sweep.py 32768 3 >> $OUT/persist.txt 2>&1
  echo "== persist=$p fusion" >> $OUT/persist.txt
  BM_GEMM_PERSIST=$p timeout 300 python tools/fusion_probe.py 8192 f32 >> $OUT/persist.txt 2>&1
done
