#!/bin/bash
# round-2: C2 (bs 1) with the pair kernel vs the 1-CTA kernel (two query tiles / one tile + two S slots)
cd $GRAFT_REPO_ROOT
for i in 1 2; do
  for e in "" "SDB_ATTN_CTA_GROUP=1" "SDB_ATTN_CTA_GROUP=1 SDB_ATTN_NT=1"; do
    env $e timeout 300 python bench.py --config c2 --no-cpu-baseline --no-e2e --steps 50 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('[$e]', round(d['value'],1), 'attn', round(d['kernels_ms']['tree_attn']*1000,1), 'accept', round(d['kernels_ms']['accept']*1000,1))"
  done
done
exit 0
