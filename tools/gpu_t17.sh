BM_GEMM_MN=1 timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "gemm and not epilogue and not fused" -p no:cacheprovider > gpurun_out/t17.txt 2>&1; echo "rc=$?" >> gpurun_out/t17.txt
for v in "BM_GEMM_MN=0" "BM_GEMM_MN=1"; do
  echo "== $v" >> gpurun_out/mn.txt
  env $v timeout 300 python tools/gemm32k_sweep.py 8192 10 >> gpurun_out/mn.txt 2>&1
done
