OUT=gpurun_out
: > $OUT/shard_lg.txt
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_dist.py tests/test_dist_device.py -x -q -m gpu -k "shard or pipelined or two_ranks or logistic" -p no:cacheprovider >> $OUT/shard_lg.txt 2>&1; echo "pytest rc=$?" >> $OUT/shard_lg.txt
BM_BENCH_SHARE_GPU=1 timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29533 bench.py --gpus 2 --steps 3 --warmup 3 > $OUT/share2_b.json 2> $OUT/share2_b.err; echo "share2 rc=$?" >> $OUT/shard_lg.txt
