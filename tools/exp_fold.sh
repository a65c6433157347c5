#!/bin/bash
# reduction timing experiments (GPU box): default, no final fold (timing only), geometry variants
for v in ${VARIANTS:-"X=1" "BM_DEBUG_NOFOLD=1"}; do
  echo "$v"; env $v timeout 120 python tools/sweep_reduce.py 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print({k:v for k,v in d.items() if k.endswith('_us') and 'cpu' not in k}, d['check'])"
done
