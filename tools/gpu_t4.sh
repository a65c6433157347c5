for v in "BM_STAGE_BATCH=4" "X=1" "BM_DEBUG_NOFOLD=1"; do
  echo "$v" >> gpurun_out/iso4.txt
  env $v timeout 200 python tools/isolated_reduce_probe.py >> gpurun_out/iso4.txt 2>&1
done
