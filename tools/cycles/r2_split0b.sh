#!/bin/bash
# adaptive first-level split: stochastic tests, C5 / C3 stochastic lines
cd $GRAFT_REPO_ROOT
O=gpurun_out
timeout -s ABRT 900 python -m pytest tests -m gpu -q -k "stochastic or lazy or c5 or validation or mixed" > $O/s0_pytest.txt 2>&1; tail -2 $O/s0_pytest.txt
j() { python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(round(d["value"],1))'; }
for rep in 1 2; do
echo "c5 $(timeout 300 python bench.py --config c5 --no-e2e --no-cpu-baseline --steps 20 | j) c3st $(timeout 300 python bench.py --mode stochastic --no-e2e --no-cpu-baseline --steps 20 | j)"
done
exit 0
