#!/bin/bash
# round-2: row stats passes through a 4 x 32 KB TMA ring -- stochastic parity, C5 lazy / eager, C3 stochastic
cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests/test_gpu_sampling.py tests/test_gpu_benched_configs.py tests/test_gpu_parity.py -m gpu -q -x -k "stoch or c5 or sampling or mss or philox or lazy or fsm or target" 2>&1 | tail -2
for i in 1 2; do
  timeout 300 python bench.py --config c5 --no-cpu-baseline --no-e2e --steps 20 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('c5 lazy', round(d['value'],1))"
  SDB_STOCH_EAGER=1 timeout 300 python bench.py --config c5 --no-cpu-baseline --no-e2e --steps 20 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('c5 eager', round(d['value'],1))"
  timeout 300 python bench.py --mode stochastic --no-cpu-baseline --no-e2e --steps 20 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('c3 stoch', round(d['value'],1), 'accept', round(d['kernels_ms']['accept']*1000,1))"
  SDB_DIAG_SKIP_VALIDATE=1 timeout 300 python bench.py --config c5 --no-cpu-baseline --no-e2e --steps 20 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('c5 chain alone', round(d['value'],1))"
done
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum --clock-control none -k regex:"row_stats|stochastic_walk" -c 14 --csv --log-file gpurun_out/r2_ring_c5.csv python bench.py --config c5 --steps 1 --warmup 3 --no-e2e --no-cpu-baseline > /dev/null 2>&1
python - <<'PY'
import csv
rows = list(csv.reader(open("gpurun_out/r2_ring_c5.csv")))
h = next(i for i, r in enumerate(rows) if "Kernel Name" in r); H = rows[h]
for r in rows[h+1:]:
    if len(r) > H.index("Metric Value") and r[H.index("Metric Name")] == "gpu__time_duration.sum":
        print(r[H.index("Kernel Name")][:30], r[H.index("Metric Value")])
PY
exit 0
