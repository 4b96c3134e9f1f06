#!/bin/bash
# persistent validation scan: finer K sweep, walk cluster width, batch dependence
cd $GRAFT_REPO_ROOT
j() { python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(round(d["value"],1))'; }
for k in 40 44 48 52 56 60; do
  echo "c5 K=$k $(SDB_VALIDATE_SMS=$k timeout 300 python bench.py --config c5 --no-e2e --no-cpu-baseline --steps 20 | j)  cl4 $(SDB_WALK_CL=4 SDB_VALIDATE_SMS=$k timeout 300 python bench.py --config c5 --no-e2e --no-cpu-baseline --steps 20 | j)"
done
for k in 40 48 56 64; do
  echo "sweep K=$k"; SDB_VALIDATE_SMS=$k timeout 600 python tools/lazy_sweep.py --batches 20,32,48,64 | python -c "
import json,sys
for l in sys.stdin: d=json.loads(l); print(d['batch'], round(d['eager_us']), round(d['lazy_us']))"
done
exit 0
