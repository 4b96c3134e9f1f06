#!/bin/bash
# round-2: C5 with the TMA-fed one-warp validation scan resident beside the lazy chain
cd $GRAFT_REPO_ROOT
for i in 1 2; do
  for v in tma old regs64; do
    lib=""; env="SDB_SCAN_TMA=1"
    [ $v = old ] && env="SDB_SCAN_TMA=0"
    [ $v = regs64 ] && lib=tools/variants/regs64/libspecdec_b200.so
    echo "== $v"
    env $env SDB_LIB=$lib timeout 300 python bench.py --config c5 --no-cpu-baseline --no-e2e --steps 20 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('c5', round(d['value'],1))"
    env $env SDB_LIB=$lib timeout 300 python bench.py --mode stochastic --no-cpu-baseline --no-e2e --steps 20 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('c3 stoch', round(d['value'],1), 'accept', round(d['kernels_ms']['accept']*1000,1))"
  done
done
timeout 900 python -m pytest tests/test_gpu_sampling.py tests/test_gpu_benched_configs.py -m gpu -q -x -k "stoch or c5 or sampling or mss or philox or lazy" 2>&1 | tail -2
exit 0
