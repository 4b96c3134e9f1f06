#!/bin/bash
# same box, interleaved: grid-stride scan (no counter, no finisher) vs counter + finisher
cd $GRAFT_REPO_ROOT
j() { python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(round(d["value"],1))'; }
for rep in 1 2 3; do
for k in 56 64; do
  echo "K=$k stride c5 $(SDB_VALIDATE_FINISH=0 SDB_VALIDATE_SMS=$k timeout 300 python bench.py --config c5 --no-e2e --no-cpu-baseline --steps 20 | j)  fin c5 $(SDB_VALIDATE_SMS=$k timeout 300 python bench.py --config c5 --no-e2e --no-cpu-baseline --steps 20 | j)"
done; done
exit 0
