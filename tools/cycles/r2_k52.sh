#!/bin/bash
# K = 52 default: stochastic tests, C5 / C3 stochastic lines
cd $GRAFT_REPO_ROOT
O=gpurun_out
timeout -s ABRT 900 python -m pytest tests -m gpu -q -k "stochastic or lazy or c5 or validation or mixed or pipeline" > $O/k52_pytest.txt 2>&1; tail -2 $O/k52_pytest.txt
for rep in 1 2; do
  timeout 300 python bench.py --config c5 --no-cpu-baseline --steps 30 > $O/k52_c5_$rep.json 2>/dev/null
  timeout 300 python bench.py --mode stochastic --no-cpu-baseline --steps 30 > $O/k52_c3st_$rep.json 2>/dev/null
  python -c "
import json
for f in ['$O/k52_c5_$rep.json','$O/k52_c3st_$rep.json']:
    d=json.load(open(f)); print(f, round(d['value'],1), round(d['roofline']['frac'],3), d['clocks']['reasons'])"
done
exit 0
