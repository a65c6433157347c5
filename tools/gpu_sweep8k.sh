for g in 2 4 6 8 12; do
  BM_GEMM_GROUP=$g timeout 120 python tools/gemm32k_sweep.py 8192 10 >> gpurun_out/sweep8k.txt 2>&1
  BM_GEMM_GROUP=$g timeout 120 python tools/gemm32k_sweep.py 16384 5 >> gpurun_out/sweep8k.txt 2>&1
done
