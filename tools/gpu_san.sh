OUT=gpurun_out
K="logistic or sum_cache or recipe or epilogue or fused_operand or fused_dim1"
timeout 1500 compute-sanitizer --tool memcheck --print-limit 10 python -m pytest tests/test_gpu_parity.py -x -q -k "$K" -p no:cacheprovider > $OUT/san_memcheck.txt 2>&1; echo "rc=$?" >> $OUT/san_memcheck.txt
timeout 1500 compute-sanitizer --tool synccheck --print-limit 10 python -m pytest tests/test_gpu_parity.py -x -q -k "logistic_accu or epilogue_bit" -p no:cacheprovider > $OUT/san_synccheck.txt 2>&1; echo "rc=$?" >> $OUT/san_synccheck.txt
timeout 1500 compute-sanitizer --tool racecheck --print-limit 10 python -m pytest tests/test_gpu_parity.py -x -q -k "logistic_accu_side_output_bit_exact and 100" -p no:cacheprovider > $OUT/san_racecheck.txt 2>&1; echo "rc=$?" >> $OUT/san_racecheck.txt
