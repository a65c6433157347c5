OUT=gpurun_out
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $OUT/smoke2.txt 2>&1; echo "smoke rc=$?" >> $OUT/smoke2.txt
timeout 900 python bench.py > $OUT/bench_n1_b.json 2> $OUT/bench_n1_b.err; echo "bench rc=$?" >> $OUT/bench_n1_b.err
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > $OUT/bench_ref_b.json 2> $OUT/bench_ref_b.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $OUT/launches_b.csv python bench.py --steps 20 --warmup 3 --no-secondary --no-cpu > /dev/null 2>&1
timeout 900 compute-sanitizer --tool memcheck --print-limit 20 python -m pytest tests/test_gpu_parity.py -x -q -k "epilogue or fused_operand or logistic_accu or sum_cache or recipe" -p no:cacheprovider > $OUT/memcheck2.txt 2>&1; echo "memcheck rc=$?" >> $OUT/memcheck2.txt
