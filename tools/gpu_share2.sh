BM_BENCH_SHARE_GPU=1 timeout 1200 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29511 bench.py --gpus 2 --steps 20 --warmup 3 --no-cpu > gpurun_out/bench_share2.json 2> gpurun_out/bench_share2.err
echo "rc=$?" >> gpurun_out/bench_share2.err
