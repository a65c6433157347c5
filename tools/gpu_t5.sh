timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "epilogue" -p no:cacheprovider > gpurun_out/t5a.txt 2>&1; echo "rc=$?" >> gpurun_out/t5a.txt
timeout 2400 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/t5.txt 2>&1; echo "rc=$?" >> gpurun_out/t5.txt
