#!/bin/bash
# reduction geometry sweep (run on the GPU box): warps mode ctas unroll
for cfg in "16 0 1 4" "16 2 1 4" "8 0 2 4" "8 2 2 4" "16 1 1 2"; do
  set -- $cfg
  BM_REDUCE_WARPS=$1 BM_REDUCE_MODE=$2 BM_REDUCE_CTAS=$3 BM_UNIT_UNROLL=$4 timeout 120 python tools/sweep_reduce.py 2>&1 | tail -1
done
