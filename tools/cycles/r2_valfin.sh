#!/bin/bash
# validation scan with the work-stealing finisher: K sweep (C5, C3 stochastic), stochastic tests, lazy crossover
cd $GRAFT_REPO_ROOT
O=gpurun_out; mkdir -p $O
j() { python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(round(d["value"],1))'; }
timeout -s ABRT 900 python -m pytest tests -m gpu -q -k "stochastic or lazy or c5 or validation" > $O/vfin_pytest.txt 2>&1; tail -2 $O/vfin_pytest.txt
for rep in 1 2; do
for k in 32 40 48 56 64; do
  echo "K=$k c5 $(SDB_VALIDATE_SMS=$k timeout 300 python bench.py --config c5 --no-e2e --no-cpu-baseline --steps 20 | j)  c3st $(SDB_VALIDATE_SMS=$k timeout 300 python bench.py --mode stochastic --no-e2e --no-cpu-baseline --steps 20 | j)"
done; done
echo "sweep default"; timeout 600 python tools/lazy_sweep.py --batches 12,16,20,24 | python -c "
import json,sys
for l in sys.stdin: d=json.loads(l); print(d['batch'], round(d['eager_us']), round(d['lazy_us']))"
exit 0
