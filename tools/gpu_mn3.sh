OUT=gpurun_out
: > $OUT/mn3.txt
timeout 2400 python -m pytest tests -m gpu -x -q -p no:cacheprovider > $OUT/final_pytest.txt 2>&1; echo "rc=$?" >> $OUT/final_pytest.txt
BM_GEMM_MN=1 timeout 1200 python -m pytest tests/test_gpu_parity.py -x -q -k "gemm or epilogue or memory_input or persistent or repeatable or random_programs" -p no:cacheprovider >> $OUT/mn3.txt 2>&1; echo "pytest MN=1 rc=$?" >> $OUT/mn3.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $OUT/final_smoke.txt 2>&1; echo "smoke rc=$?" >> $OUT/final_smoke.txt
timeout 900 python bench.py > $OUT/final_bench.json 2> $OUT/final_bench.err; echo "bench rc=$?" >> $OUT/final_bench.err
