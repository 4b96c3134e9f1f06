#!/bin/bash
# round-2: row stats HBM pass -- L2 bulk prefetch on/off, 4 or 8 loads in flight per thread
cd $GRAFT_REPO_ROOT
for i in 1 2; do
  for v in base nopf ku8 ku8nopf; do
    lib=""; [ $v != base ] && lib=tools/variants/$v/libspecdec_b200.so
    SDB_LIB=$lib timeout 300 python bench.py --config c5 --no-cpu-baseline --no-e2e --steps 20 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$v c5 lazy', round(d['value'],1))"
    SDB_LIB=$lib SDB_DIAG_SKIP_VALIDATE=1 timeout 300 python bench.py --config c5 --no-cpu-baseline --no-e2e --steps 20 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$v c5 chain', round(d['value'],1))"
    SDB_LIB=$lib SDB_STOCH_EAGER=1 timeout 300 python bench.py --config c5 --no-cpu-baseline --no-e2e --steps 20 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$v c5 eager', round(d['value'],1))"
  done
done
exit 0
