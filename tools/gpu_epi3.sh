OUT=gpurun_out
: > $OUT/epi3.txt
timeout 1200 python -m pytest tests/test_gpu_parity.py -x -q -k "gemm or epilogue or memory_input or persistent" -p no:cacheprovider >> $OUT/epi3.txt 2>&1; echo "pytest rc=$?" >> $OUT/epi3.txt
BM_GEMM_PERSIST=1 timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -k "memory_input" -p no:cacheprovider >> $OUT/epi3.txt 2>&1; echo "pytest persist rc=$?" >> $OUT/epi3.txt
timeout 300 python tools/epi_mem_probe.py 8192 8 >> $OUT/epi3.txt 2>&1
timeout 300 python tools/fusion_probe.py 8192 f32 >> $OUT/epi3.txt 2>&1
