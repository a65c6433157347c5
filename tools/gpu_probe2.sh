set -x
OUT=gpurun_out
timeout 300 python tools/cfg5_overhead_probe.py > $OUT/cfg5_probe.txt 2>&1
nvidia-smi --query-gpu=index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap --format=csv -lms 100 > $OUT/clocks_gemm32k.csv &
SMI=$!
BM_GEMM_KPASS=8192 timeout 300 python tools/gemm32k_sweep.py 32768 5 > $OUT/gemm32k.txt 2>&1
kill $SMI
for t in logistic_fused:bm_lgrad gemm32k_f32:gemm_3xtf32_pair cfg1:bm_reduce; do
  w=${t%%:*}; k=${t##*:}
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:$k -s 1 -c 1 \
      -o $OUT/prof_$w python tools/profile_targets.py $w > $OUT/ncu_$w.log 2>&1
done
ls -la $OUT
