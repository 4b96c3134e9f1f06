#!/bin/bash
# claimed-ahead row counter; finisher on/off; K sweep
cd $GRAFT_REPO_ROOT
j() { python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(round(d["value"],1))'; }
for rep in 1 2; do
for k in 48 56 64; do
  echo "K=$k fin c5 $(SDB_VALIDATE_SMS=$k timeout 300 python bench.py --config c5 --no-e2e --no-cpu-baseline --steps 20 | j)  nofin c5 $(SDB_VALIDATE_FINISH=0 SDB_VALIDATE_SMS=$k timeout 300 python bench.py --config c5 --no-e2e --no-cpu-baseline --steps 20 | j) fin c3st $(SDB_VALIDATE_SMS=$k timeout 300 python bench.py --mode stochastic --no-e2e --no-cpu-baseline --steps 20 | j)"
done; done
exit 0
