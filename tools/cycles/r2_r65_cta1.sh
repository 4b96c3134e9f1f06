#!/bin/bash
# round-2: R = 65 / R = 64 with the 1-CTA kernel (one query tile, two S slots) vs the pair kernel
cd $GRAFT_REPO_ROOT
for t in 65 64; do
  for e in "" "SDB_ATTN_CTA_GROUP=1 SDB_ATTN_NT=1" "SDB_ATTN_CTA_GROUP=1"; do
    env $e timeout 300 python bench.py --tree $t --no-cpu-baseline --no-e2e --steps 20 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('tree $t [$e]', round(d['value'],1), 'attn', round(d['kernels_ms']['tree_attn']*1000,1))"
  done
done
exit 0
