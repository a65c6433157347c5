# ncu after the barrier-scope fix: plain pair GEMM 8192^3 and the exp - C fused epilogue
OUT=gpurun_out
timeout 600 ncu --set full --clock-control none --import-source on -k regex:gemm_3xtf32_pair -s 1 -c 1 \
    -o $OUT/prof_gemm_f32_fix python tools/profile_targets.py gemm_f32 > $OUT/ncu_gemm_f32_fix.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:bm_gemm_epi -s 1 -c 1 \
    -o $OUT/prof_epi_exp_minus_c_fix python tools/profile_targets.py epi_exp_minus_c > $OUT/ncu_epi_fix.log 2>&1
