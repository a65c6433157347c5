OUT=gpurun_out
timeout 1200 compute-sanitizer --tool memcheck --print-limit 10 python -m pytest tests/test_gpu_parity.py -x -q -k "memory_input or persistent or epilogue_bit or gemm_shapes" -p no:cacheprovider > $OUT/san2_memcheck.txt 2>&1; echo "memcheck rc=$?" >> $OUT/san2_memcheck.txt
timeout 1200 compute-sanitizer --tool racecheck --print-limit 10 python -m pytest tests/test_gpu_parity.py -x -q -k "memory_input and 1024-768" -p no:cacheprovider > $OUT/san2_racecheck.txt 2>&1; echo "racecheck rc=$?" >> $OUT/san2_racecheck.txt
timeout 1200 compute-sanitizer --tool synccheck --print-limit 10 python -m pytest tests/test_gpu_parity.py -x -q -k "memory_input and 1024-768" -p no:cacheprovider > $OUT/san2_synccheck.txt 2>&1; echo "synccheck rc=$?" >> $OUT/san2_synccheck.txt
