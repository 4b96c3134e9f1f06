#!/bin/bash
# K sweep with the unsplit first level (C5), interleaved
cd $GRAFT_REPO_ROOT
j() { python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(round(d["value"],1))'; }
for rep in 1 2; do
  for k in 46 50 52 54 58; do echo "rep $rep K=$k c5 $(SDB_VALIDATE_SMS=$k timeout 300 python bench.py --config c5 --no-e2e --no-cpu-baseline --steps 20 | j)"; done
done
exit 0
