for b in 128 64 32; do
  echo "== boxc $b" >> gpurun_out/lgbox.txt
  BM_LG_BOXC=$b timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -k "logistic" -p no:cacheprovider 2>&1 | tail -1 >> gpurun_out/lgbox.txt
  BM_LG_BOXC=$b timeout 300 python tools/cfg5_timeline_probe.py >> gpurun_out/lgbox.txt 2>&1
  BM_LG_BOXC=$b timeout 300 python tools/lgrad_k_probe.py 1024 >> gpurun_out/lgbox.txt 2>&1
done
