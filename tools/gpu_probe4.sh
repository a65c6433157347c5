OUT=gpurun_out
timeout 300 python tools/isolated_reduce_probe.py > $OUT/iso3.txt 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -s 120 -c 40 --csv --log-file $OUT/cfg5_launches.csv python tools/cfg5_timeline_probe.py > /dev/null 2>&1
