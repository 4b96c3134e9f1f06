#!/bin/bash
# round-2: lazy chain row stats split over 2-CTA clusters (SDB_ST_SPLIT=1) vs one CTA per row
cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests/test_gpu_sampling.py tests/test_gpu_benched_configs.py -m gpu -q -x -k "stoch or c5 or sampling or mss or philox or lazy or fsm or target" 2>&1 | tail -2
for i in 1 2; do
  for e in 4 2 1; do
    SDB_ST_SPLIT=$e timeout 300 python bench.py --config c5 --no-cpu-baseline --no-e2e --steps 20 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('split=$e c5', round(d['value'],1))"
    SDB_ST_SPLIT=$e timeout 300 python bench.py --mode stochastic --no-cpu-baseline --no-e2e --steps 20 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('split=$e c3 stoch', round(d['value'],1), 'accept', round(d['kernels_ms']['accept']*1000,1))"
    SDB_ST_SPLIT=$e SDB_DIAG_SKIP_VALIDATE=1 timeout 300 python bench.py --config c5 --no-cpu-baseline --no-e2e --steps 20 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('split=$e c5 chain alone', round(d['value'],1))"
  done
done
exit 0
