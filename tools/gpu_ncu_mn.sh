OUT=gpurun_out
timeout 600 ncu --set full --clock-control none --import-source on -k regex:gemm_3xtf32_pair -s 1 -c 1 \
    -o $OUT/prof_gemm_f32_mn python tools/profile_targets.py gemm_f32 > $OUT/ncu_gemm_f32_mn.log 2>&1
