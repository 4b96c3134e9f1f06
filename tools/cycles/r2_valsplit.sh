#!/bin/bash
# persistent scan K x chain shape (row split 1 / 2 CTAs, walk cluster 8 / 4) at C5
cd $GRAFT_REPO_ROOT
j() { python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(round(d["value"],1))'; }
for k in 48 56 64; do
  echo "K=$k split2 $(SDB_VALIDATE_SMS=$k timeout 300 python bench.py --config c5 --no-e2e --no-cpu-baseline --steps 20 | j) split1 $(SDB_ST_SPLIT=1 SDB_VALIDATE_SMS=$k timeout 300 python bench.py --config c5 --no-e2e --no-cpu-baseline --steps 20 | j) diag-noscan $(SDB_DIAG_SKIP_VALIDATE=1 SDB_VALIDATE_SMS=$k timeout 300 python bench.py --config c5 --no-e2e --no-cpu-baseline --steps 20 | j)"
done
exit 0
