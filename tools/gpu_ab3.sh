# A/B: bm_lgrad z-exchange wait at cluster scope (old) vs CTA scope (head)
OUT=gpurun_out
L=paper_2308_03120_b200/libb200mat.so
: > $OUT/ab3.txt
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_baseline_shapes.py -x -q -k "logistic or lgrad" -p no:cacheprovider >> $OUT/ab3.txt 2>&1; echo "pytest head rc=$?" >> $OUT/ab3.txt
for round in 1 2 3; do
for v in old head; do
  cp abtmp/lib_$v.so $L; touch $L
  echo "== $v" >> $OUT/ab3.txt
  timeout 300 python tools/cfg5_timeline_probe.py >> $OUT/ab3.txt 2>&1
done
done
cp abtmp/lib_head.so $L
