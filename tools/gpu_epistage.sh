OUT=gpurun_out
: > $OUT/epistage.txt
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "memory_input or epilogue or persistent" -p no:cacheprovider >> $OUT/epistage.txt 2>&1; echo "pytest rc=$?" >> $OUT/epistage.txt
for st in 1 0 1 0; do
  echo "== stage=$st" >> $OUT/epistage.txt
  BM_GEMM_EPI_STAGE=$st timeout 300 python tools/epi_mem_probe.py 8192 8 >> $OUT/epistage.txt 2>&1
done
timeout 300 compute-sanitizer --tool memcheck --print-limit 10 python -m pytest tests/test_gpu_parity.py -x -q -k "memory_input" -p no:cacheprovider > $OUT/epistage_memcheck.txt 2>&1; echo "memcheck rc=$?" >> $OUT/epistage_memcheck.txt
