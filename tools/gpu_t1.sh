timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "logistic or sum_cache" -p no:cacheprovider > gpurun_out/t1.txt 2>&1; echo "rc=$?" >> gpurun_out/t1.txt
timeout 300 python tools/cfg5_timeline_probe.py > gpurun_out/cfg5_timeline2.txt 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -s 60 -c 30 --csv --log-file gpurun_out/cfg5_launches2.csv python tools/cfg5_timeline_probe.py > /dev/null 2>&1
