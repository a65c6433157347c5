timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "fused_operand or epilogue or gemm" -p no:cacheprovider > gpurun_out/t6.txt 2>&1; echo "rc=$?" >> gpurun_out/t6.txt
