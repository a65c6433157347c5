BM_GEMM_CONV=1 timeout 300 python -m pytest tests/test_gpu_parity.py -x -q -k "gemm and not epilogue and not fused and not 32768" -p no:cacheprovider > gpurun_out/t20.txt 2>&1; echo "rc=$?" >> gpurun_out/t20.txt
for v in "BM_GEMM_CONV=0" "BM_GEMM_CONV=1"; do
  echo "== $v" >> gpurun_out/conv.txt
  env $v timeout 120 python tools/gemm32k_sweep.py 8192 10 >> gpurun_out/conv.txt 2>&1
  env $v timeout 120 python tools/gemm32k_sweep.py 16384 5 >> gpurun_out/conv.txt 2>&1
  env $v timeout 200 python tools/gemm32k_sweep.py 32768 3 >> gpurun_out/conv.txt 2>&1
done
