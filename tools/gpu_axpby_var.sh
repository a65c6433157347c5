OUT=gpurun_out
: > $OUT/axv.txt
for i in 1 2 3 4; do timeout 300 python tools/epi_mem_probe.py 8192 10 >> $OUT/axv.txt 2>&1; done
