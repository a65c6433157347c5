OUT=gpurun_out
timeout 2400 python -m pytest tests -m gpu -x -q -p no:cacheprovider > $OUT/t9.txt 2>&1; echo "rc=$?" >> $OUT/t9.txt
timeout 300 python tools/cfg5_timeline_probe.py > $OUT/cfg5_timeline5.txt 2>&1
for t in logistic_fused:bm_lgrad rdim0:rdim0_cta; do
  w=${t%%:*}; k=${t##*:}
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:$k -s 1 -c 1 -o $OUT/prof2_$w python tools/profile_targets.py $w > $OUT/ncu2_$w.log 2>&1
done
