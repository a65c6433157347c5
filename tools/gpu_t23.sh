BM_GEMM_CONV=1 timeout 600 ncu --set full --clock-control none -k regex:gemm_3xtf32_conv -s 1 -c 1 -o gpurun_out/prof_conv python tools/gemm32k_sweep.py 8192 2 > gpurun_out/ncu_conv.log 2>&1
