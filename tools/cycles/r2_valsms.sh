#!/bin/bash
# C5 / C3 stochastic: validation scan as a persistent K-SM kernel (SDB_VALIDATE_SMS=K) vs the one-row low-priority CTAs
cd $GRAFT_REPO_ROOT
O=gpurun_out; mkdir -p $O
j() { python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(round(d["value"],1), {k: round(v*1000,1) for k,v in d["kernels_ms"].items()})'; }
for rep in 1 2; do
for k in 0 48 64 80 96 112; do
  echo "c5 K=$k $(SDB_VALIDATE_SMS=$k timeout 300 python bench.py --config c5 --no-e2e --no-cpu-baseline --steps 20 | j)"
done
done
for k in 0 64 80; do
  echo "c3st K=$k $(SDB_VALIDATE_SMS=$k timeout 300 python bench.py --mode stochastic --no-e2e --no-cpu-baseline --steps 20 | j)"
done
SDB_VALIDATE_SMS=80 timeout -s ABRT 900 python -m pytest tests -m gpu -q -k "stochastic or lazy or c5 or nan" > $O/vs_pytest.txt 2>&1; tail -2 $O/vs_pytest.txt
exit 0
