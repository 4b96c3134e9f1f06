#!/bin/bash
# round-2: 16-lane half-row softmax for warps with <= 16 live rows (R = 65 tail) -- parity, A/B
cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_benched_configs.py -m gpu -q -x -k "tcgen05 or r65 or draft or bench_step or irope or golden or c4" 2>&1 | tail -2
for i in 1 2; do
  for v in new pre16; do
    lib=""; [ $v = pre16 ] && lib=tools/variants/pre16/libspecdec_b200.so
    SDB_LIB=$lib timeout 300 python bench.py --tree 65 --no-cpu-baseline --no-e2e --steps 20 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$v r65 step', round(d['value'],1), 'attn', round(d['kernels_ms']['tree_attn']*1000,1))"
    SDB_LIB=$lib timeout 300 python bench.py --no-cpu-baseline --no-e2e --steps 20 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$v c3 step', round(d['value'],1), 'attn', round(d['kernels_ms']['tree_attn']*1000,1))"
  done
done
exit 0
