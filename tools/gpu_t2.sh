timeout 2400 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/t2.txt 2>&1; echo "rc=$?" >> gpurun_out/t2.txt
timeout 300 python tools/cfg5_timeline_probe.py > gpurun_out/cfg5_timeline3.txt 2>&1
timeout 300 python tools/host_breakdown_probe.py > gpurun_out/host_breakdown2.txt 2>&1
