OUT=gpurun_out
for w in epi_exp epi_exp_minus_c; do
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:bm_gemm_epi -s 1 -c 1 \
      -o $OUT/prof_$w python tools/profile_targets.py $w > $OUT/ncu_$w.log 2>&1
done
