echo "== noconvert" >> gpurun_out/conv3.txt
BM_GEMM_CONV=1 timeout 120 python tools/gemm32k_sweep.py 8192 10 >> gpurun_out/conv3.txt 2>&1
