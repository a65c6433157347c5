# A/B: DMMA GEMM with 4 warps of 32x64 (old) vs 8 warps of 32x32 (head) per 64x128 CTA
OUT=gpurun_out
L=paper_2308_03120_b200/libb200mat.so
: > $OUT/ab5.txt
cp abtmp/lib_head.so $L; touch $L
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "gemm and (f64 or float64 or dt1 or vs_reference or shapes or trans)" -p no:cacheprovider >> $OUT/ab5.txt 2>&1; echo "pytest head rc=$?" >> $OUT/ab5.txt
for round in 1 2; do
for v in old head; do
  cp abtmp/lib_$v.so $L; touch $L
  echo "== $v" >> $OUT/ab5.txt
  timeout 300 python tools/fusion_probe.py 8192 f64 >> $OUT/ab5.txt 2>&1
done
done
cp abtmp/lib_head.so $L
