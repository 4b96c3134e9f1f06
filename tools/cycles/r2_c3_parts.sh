#!/bin/bash
# C3: attention alone on 64 / 74 CTA pairs vs the full step (where the step's last ~25 us go)
cd $GRAFT_REPO_ROOT
for c in 64 74; do echo "attn ctas=$c $(timeout 300 python tools/attn_bench.py c3 --ctas $c | cut -c1-110)"; done
echo "step $(timeout 300 python bench.py --no-e2e --no-cpu-baseline --steps 30 | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(round(d["value"],1), d["kernels_ms"])')"
exit 0
