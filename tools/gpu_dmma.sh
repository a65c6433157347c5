# DMMA issue ceiling + ncu of the f64 GEMM at 8192^3
OUT=gpurun_out
timeout 120 ./tools/dmma_peak > $OUT/dmma_peak.txt 2>&1
nvidia-smi --query-gpu=clocks.sm,power.draw,clocks_event_reasons.active --format=csv,noheader -lms 100 > $OUT/dmma_clk.csv &
SMI=$!
timeout 120 ./tools/dmma_peak >> $OUT/dmma_peak.txt 2>&1
kill $SMI
timeout 600 ncu --set full --clock-control none --import-source on -k regex:gemm_dmma -s 1 -c 1 \
    -o $OUT/prof_gemm_f64 python tools/profile_targets.py gemm_f64 > $OUT/ncu_gemm_f64.log 2>&1
