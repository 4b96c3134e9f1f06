#!/bin/bash
# C2 (bs 1) step vs attention worker count (num_splits = CTA-pair workers; 0 = auto)
O=gpurun_out; T=${1:-c2}; mkdir -p $O
for s in ${SPLITS:-0 16 24 32 48 64 74}; do
  echo "== splits $s"
  timeout 300 python bench.py --config c2 --splits $s --no-cpu-baseline --no-e2e 2>>$O/${T}.err | grep -o '"value": [0-9.]*\|"kernels_ms": {[^}]*}'
done
exit 0
