#!/bin/bash
# round-2: pair kernel -- rotating TMEM roles (+ next-unit Q L2 prefetch) vs HEAD
cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_benched_configs.py -m gpu -q -x -k "tcgen05 or draft or irope or golden or bench_step or c4 or max_ctx or other_trees or r65" 2>&1 | tail -2
TRACE_ROWS=62,63,64,65,66,67,68 SDB_LIB=paper_2508_08192_b200/_lib/libspecdec_b200_trace.so timeout 120 python tools/trace_attn.py c3 2>&1 | grep -A8 "^item:"
for i in 1 2 3; do
  for v in new roles preepi; do
    lib=""; [ $v != new ] && lib=tools/variants/$v/libspecdec_b200.so
    SDB_LIB=$lib timeout 120 python tools/attn_bench.py c3 --iters 10 --reps 5 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$v', round(d['ms']*1000,1))"
  done
done
for v in new preepi; do
  lib=""; [ $v != new ] && lib=tools/variants/$v/libspecdec_b200.so
  SDB_LIB=$lib timeout 300 python bench.py --no-cpu-baseline --no-e2e --steps 30 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$v step', round(d['value'],1))"
  SDB_LIB=$lib timeout 300 python bench.py --config c4 --steps 5 --no-cpu-baseline --no-e2e | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$v c4 step', round(d['value'],1))"
done
exit 0
