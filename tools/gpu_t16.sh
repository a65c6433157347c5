timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "recipe" -p no:cacheprovider > gpurun_out/t16.txt 2>&1; echo "rc=$?" >> gpurun_out/t16.txt
