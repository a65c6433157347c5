L=paper_2308_03120_b200/libb200mat.so
for round in 1 2; do
for v in old head; do
  cp gpurun_out/ab/lib_$v.so $L; touch $L
  echo "== $v" >> gpurun_out/ab.txt
  timeout 120 python tools/gemm32k_sweep.py 8192 10 >> gpurun_out/ab.txt 2>&1
done
done
for v in old head; do
  cp gpurun_out/ab/lib_$v.so $L; touch $L
  echo "== $v 32k" >> gpurun_out/ab.txt
  timeout 200 python tools/gemm32k_sweep.py 32768 3 >> gpurun_out/ab.txt 2>&1
done
rm -rf gpurun_out/ab
