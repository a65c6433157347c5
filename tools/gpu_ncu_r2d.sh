# ncu at the end of round 2: persistent pair GEMM (raster group 8) and the staged 2AB^T + 3C epilogue
OUT=gpurun_out
timeout 600 ncu --set full --clock-control none --import-source on -k regex:gemm_3xtf32_pair -s 1 -c 1 \
    -o $OUT/prof_gemm_f32_final python tools/profile_targets.py gemm_f32 > $OUT/ncu_gemm_f32_final.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:bm_gemm_epi -s 1 -c 1 \
    -o $OUT/prof_epi_axpby_final python tools/profile_targets.py epi_axpby > $OUT/ncu_epi_axpby_final.log 2>&1
