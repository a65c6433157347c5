timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "logistic" -p no:cacheprovider > gpurun_out/t11.txt 2>&1; echo "rc=$?" >> gpurun_out/t11.txt
BM_DEBUG_LGRAD=1 timeout 600 python tools/lgrad_k_probe.py 1024 2048 4096 > gpurun_out/lgrad_k.txt 2>&1
