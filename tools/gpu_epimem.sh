OUT=gpurun_out
: > $OUT/epimem.txt
BM_GEMM_PERSIST=1 timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "persistent_pairs" -p no:cacheprovider >> $OUT/epimem.txt 2>&1; echo "pytest rc=$?" >> $OUT/epimem.txt
for p in 1 0 1 0; do
  BM_GEMM_PERSIST=$p timeout 300 python tools/epi_mem_probe.py 8192 8 >> $OUT/epimem.txt 2>&1
done
