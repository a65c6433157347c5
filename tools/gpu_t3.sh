timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "logistic or sum_cache or recipe" -p no:cacheprovider > gpurun_out/t3.txt 2>&1; echo "rc=$?" >> gpurun_out/t3.txt
timeout 300 python tools/cfg5_timeline_probe.py > gpurun_out/cfg5_timeline4.txt 2>&1
BM_PLAN_CACHE=0 timeout 300 python tools/cfg5_timeline_probe.py >> gpurun_out/cfg5_timeline4.txt 2>&1
