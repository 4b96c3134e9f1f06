#!/bin/bash
# lazy chain: first level without the 2-CTA row split (SDB_ST_SPLIT0=1), K 44..56
cd $GRAFT_REPO_ROOT
j() { python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(round(d["value"],1))'; }
for rep in 1 2; do
for k in 44 50 56; do
  echo "K=$k c5 split0=2 $(SDB_VALIDATE_SMS=$k timeout 300 python bench.py --config c5 --no-e2e --no-cpu-baseline --steps 20 | j) split0=1 $(SDB_ST_SPLIT0=1 SDB_VALIDATE_SMS=$k timeout 300 python bench.py --config c5 --no-e2e --no-cpu-baseline --steps 20 | j) all1 $(SDB_ST_SPLIT=1 SDB_VALIDATE_SMS=$k timeout 300 python bench.py --config c5 --no-e2e --no-cpu-baseline --steps 20 | j)"
done; done
echo "c3st split0=2 $(timeout 300 python bench.py --mode stochastic --no-e2e --no-cpu-baseline --steps 20 | j) split0=1 $(SDB_ST_SPLIT0=1 timeout 300 python bench.py --mode stochastic --no-e2e --no-cpu-baseline --steps 20 | j)"
exit 0
