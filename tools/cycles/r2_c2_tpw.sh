#!/bin/bash
# C2 (bs 1): target tiles per attention worker (SDB_ATTN_TPW, default 9), interleaved
cd $GRAFT_REPO_ROOT
j() { python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(round(d["value"],1), round(d["kernels_ms"]["tree_attn"]*1e3,1))'; }
for rep in 1 2; do
  for t in 5 7 9 12 16 24; do
    echo "rep $rep tpw $t: $(SDB_ATTN_TPW=$t timeout 300 python bench.py --config c2 --no-e2e --no-cpu-baseline --steps 50 | j)"
  done
done
exit 0
