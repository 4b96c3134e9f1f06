#!/bin/bash
# C3 greedy: reserve sweep (SMs left to the concurrent scan), interleaved
cd $GRAFT_REPO_ROOT
j() { python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(round(d["value"],1))'; }
for rep in 1 2; do
  for k in 16 18 20 22 24; do
    echo "rep $rep reserve $k: $(SDB_RESERVE_SMS=$k timeout 300 python bench.py --no-e2e --no-cpu-baseline --steps 30 | j)"
  done
done
exit 0
