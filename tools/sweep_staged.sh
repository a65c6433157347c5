#!/bin/bash
# staged-accu sweep (GPU box): legacy path vs staged with several consumer counts
BM_STAGED=0 timeout 120 python tools/sweep_reduce.py 2>&1 | tail -1
for c in ${CONSUMERS:-4 6 8}; do
  echo "consumers=$c"; BM_STAGED_CONSUMERS=$c timeout 120 python tools/sweep_reduce.py 2>&1 | tail -1
done
