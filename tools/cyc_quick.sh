#!/bin/bash
# quick check: gpu tests + C2/C3 (+ optional extra bench args) summary lines
timeout 900 python -m pytest tests -q -m gpu -x 2>&1 | tail -2
for c in "$@"; do python bench.py $c --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['config']['workload'], round(d['value'],1), {k: round(v*1e3,1) for k,v in d['kernels_ms'].items()}, round(d['roofline']['frac'],3), round(d['e2e']['value'],1))"; done
exit 0
