BM_GEMM_CONV=1 timeout 300 python -m pytest tests/test_gpu_parity.py -x -q -k "gemm and not epilogue and not fused and not 32768" -p no:cacheprovider > gpurun_out/t21.txt 2>&1; echo "rc=$?" >> gpurun_out/t21.txt
for v in "BM_GEMM_CONV=1"; do
  echo "== $v" >> gpurun_out/conv2.txt
  env $v timeout 120 python tools/gemm32k_sweep.py 8192 10 >> gpurun_out/conv2.txt 2>&1
done
