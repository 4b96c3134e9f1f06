#!/bin/bash
# e2e through HostStepPipeline: tests, chunk sweep on the default bench (C3) and stochastic
cd $GRAFT_REPO_ROOT
O=gpurun_out; mkdir -p $O
timeout -s ABRT 600 python -m pytest tests/test_gpu_host_pipeline.py -q -x > $O/pipe_pytest.txt 2>&1; tail -3 $O/pipe_pytest.txt
e() { python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(round(d["value"],1), d["e2e"])'; }
for c in 1 2 4 8; do
  echo "chunks=$c $(SDB_E2E_CHUNKS=$c timeout 400 python bench.py --no-cpu-baseline --steps 20 | e)"
done
for c in 1 4; do
  echo "stoch chunks=$c $(SDB_E2E_CHUNKS=$c timeout 400 python bench.py --mode stochastic --no-cpu-baseline --steps 20 | e)"
done
exit 0
