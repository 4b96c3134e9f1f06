#!/bin/bash
# lazy chain as programmatic dependent launches: tests, A/B (SDB_CHAIN_PDL=0), interleaved
cd $GRAFT_REPO_ROOT
O=gpurun_out; mkdir -p $O
timeout -s ABRT 900 python -m pytest tests -m gpu -q -k "stochastic or lazy or c5 or validation or mixed or pipeline" > $O/cpdl_pytest.txt 2>&1; tail -2 $O/cpdl_pytest.txt
j() { python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(round(d["value"],1))'; }
for rep in 1 2 3; do
  echo "c5 pdl $(timeout 300 python bench.py --config c5 --no-e2e --no-cpu-baseline --steps 20 | j) nopdl $(SDB_CHAIN_PDL=0 timeout 300 python bench.py --config c5 --no-e2e --no-cpu-baseline --steps 20 | j)  c3st pdl $(timeout 300 python bench.py --mode stochastic --no-e2e --no-cpu-baseline --steps 20 | j) nopdl $(SDB_CHAIN_PDL=0 timeout 300 python bench.py --mode stochastic --no-e2e --no-cpu-baseline --steps 20 | j)"
done
echo "chain alone: pdl $(SDB_DIAG_SKIP_VALIDATE=1 timeout 300 python bench.py --config c5 --no-e2e --no-cpu-baseline --steps 20 | j) nopdl $(SDB_CHAIN_PDL=0 SDB_DIAG_SKIP_VALIDATE=1 timeout 300 python bench.py --config c5 --no-e2e --no-cpu-baseline --steps 20 | j)"
exit 0
