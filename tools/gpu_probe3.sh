OUT=gpurun_out
timeout 300 python tools/cfg5_timeline_probe.py > $OUT/cfg5_timeline.txt 2>&1
for v in "X=1" "BM_DEBUG_NOFOLD=1" "BM_GRAB_BYTES=8192" "BM_GRAB_BYTES=4096" "BM_REDUCE_WARPS=16" "BM_REDUCE_WARPS=8"; do
  echo "$v" >> $OUT/iso.txt
  env $v timeout 200 python tools/isolated_reduce_probe.py >> $OUT/iso.txt 2>&1
done
