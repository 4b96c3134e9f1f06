#!/bin/bash
# flat-stream validation scan (row list in shared memory): tests, K sweep, ncu of the scan alone
cd $GRAFT_REPO_ROOT
O=gpurun_out; mkdir -p $O
j() { python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(round(d["value"],1))'; }
timeout -s ABRT 900 python -m pytest tests -m gpu -q -k "stochastic or lazy or c5 or validation" > $O/vflat_pytest.txt 2>&1; tail -2 $O/vflat_pytest.txt
for k in 36 40 44 48 56; do
  echo "K=$k c5 $(SDB_VALIDATE_SMS=$k timeout 300 python bench.py --config c5 --no-e2e --no-cpu-baseline --steps 20 | j) c3st $(SDB_VALIDATE_SMS=$k timeout 300 python bench.py --mode stochastic --no-e2e --no-cpu-baseline --steps 20 | j)"
done
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum --clock-control none -k regex:stochastic_validate_persistent -c 2 python bench.py --config c5 --steps 1 --warmup 3 --no-e2e --no-cpu-baseline 2>&1 | grep -E "duration|dram__bytes" | head -4
exit 0
