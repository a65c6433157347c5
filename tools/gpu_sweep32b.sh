for r in 1 2; do for g in 4 6; do
  BM_GEMM_GROUP=$g timeout 200 python tools/gemm32k_sweep.py 32768 3 >> gpurun_out/sweep32b.txt 2>&1
  BM_GEMM_GROUP=$g timeout 120 python tools/gemm32k_sweep.py 16384 5 >> gpurun_out/sweep32b.txt 2>&1
done; done
