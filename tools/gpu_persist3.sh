# persistent pairs on by default: parity, then persist 0/1 interleaved
OUT=gpurun_out
: > $OUT/persist3.txt
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_baseline_shapes.py -x -q -k "gemm or epilogue or memory_input or persistent or repeatable" -p no:cacheprovider >> $OUT/persist3.txt 2>&1; echo "pytest rc=$?" >> $OUT/persist3.txt
for round in 1 2 3; do
for p in 0 1; do
  for n in 8192 16384; do
    echo "persist=$p" >> $OUT/persist3.txt
    BM_GEMM_PERSIST=$p timeout 200 python tools/gemm32k_sweep.py $n 10 >> $OUT/persist3.txt 2>&1
  done
done
done
for p in 0 1; do
  echo "persist=$p" >> $OUT/persist3.txt
  BM_GEMM_PERSIST=$p timeout 300 python tools/gemm32k_sweep.py 32768 3 >> $OUT/persist3.txt 2>&1
  BM_GEMM_PERSIST=$p timeout 300 python tools/fusion_probe.py 8192 f32 >> $OUT/persist3.txt 2>&1
done
