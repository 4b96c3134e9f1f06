#!/bin/bash
# round-2: R = 65 tail rows fused into the last row block's units (warps 2 / 3) -- parity, then A/B vs the padded block
cd $GRAFT_REPO_ROOT
timeout 300 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "fused_tail" 2>&1 | tail -15
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_benched_configs.py -m gpu -q -x -k "tcgen05 or r65 or draft or bench_step or irope or golden or c4 or 65" 2>&1 | tail -4
for i in 1 2; do
  for t in 1 0; do  # (SDB_ATTN_TAIL: 1 fused tail rows, 0 padded row block = default)
    SDB_ATTN_TAIL=$t timeout 300 python bench.py --tree 65 --no-cpu-baseline --no-e2e --steps 20 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('tail=$t r65 step', round(d['value'],1), 'attn', round(d['kernels_ms']['tree_attn']*1000,1))"
  done
  timeout 300 python bench.py --no-cpu-baseline --no-e2e --steps 20 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('c3 step', round(d['value'],1), 'attn', round(d['kernels_ms']['tree_attn']*1000,1))"
done
exit 0
