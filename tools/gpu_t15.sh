timeout 2400 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/t15.txt 2>&1; echo "rc=$?" >> gpurun_out/t15.txt
