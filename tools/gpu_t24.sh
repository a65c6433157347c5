for v in "X=1" "BM_DEBUG_EXTFOLD=1"; do
  echo "== $v" >> gpurun_out/iso5.txt
  env $v timeout 200 python tools/isolated_reduce_probe.py >> gpurun_out/iso5.txt 2>&1
done
