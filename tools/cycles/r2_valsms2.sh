#!/bin/bash
# persistent validation scan: K x unroll sweep (C5, C3 stochastic), lazy/eager crossover with it
cd $GRAFT_REPO_ROOT
j() { python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(round(d["value"],1), {k: round(v*1000,1) for k,v in d["kernels_ms"].items()})'; }
for u in 8 12; do for k in 56 64 72; do
  echo "c5 U=$u K=$k $(SDB_VALIDATE_UNROLL=$u SDB_VALIDATE_SMS=$k timeout 300 python bench.py --config c5 --no-e2e --no-cpu-baseline --steps 20 | j)"
done; done
for k in 40 48 56 64 72; do
  echo "c3st K=$k $(SDB_VALIDATE_SMS=$k timeout 300 python bench.py --mode stochastic --no-e2e --no-cpu-baseline --steps 20 | j)"
done
echo "sweep K=0";  timeout 600 python tools/lazy_sweep.py --batches 16,24,32,48
echo "sweep K=64"; SDB_VALIDATE_SMS=64 timeout 600 python tools/lazy_sweep.py --batches 16,24,32,48
exit 0
