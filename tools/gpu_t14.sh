timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "gemm or epilogue or logistic" -p no:cacheprovider > gpurun_out/t14.txt 2>&1; echo "rc=$?" >> gpurun_out/t14.txt
for v in "BM_GEMM_PERSIST=0" "X=1"; do
  echo "== $v" >> gpurun_out/persist.txt
  env $v timeout 300 python tools/gemm32k_sweep.py 8192 10 >> gpurun_out/persist.txt 2>&1
  env $v timeout 300 python tools/gemm32k_sweep.py 16384 5 >> gpurun_out/persist.txt 2>&1
  env $v timeout 300 python tools/gemm32k_sweep.py 32768 3 >> gpurun_out/persist.txt 2>&1
  env $v timeout 600 python tools/fusion_probe.py 8192 f32 >> gpurun_out/persist.txt 2>&1
done
