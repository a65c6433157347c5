timeout 300 python tools/cfg5_timeline_probe.py > gpurun_out/cfg5_timeline6.txt 2>&1
timeout 300 python tools/host_breakdown_probe.py > gpurun_out/host_breakdown3.txt 2>&1
