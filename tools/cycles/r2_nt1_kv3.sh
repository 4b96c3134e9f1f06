#!/bin/bash
# round-2: 1-CTA kernel with a two S slots + fixed reference (one query tile) -- parity, chain-3 / N8 A/B, draft round
cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_benched_configs.py -m gpu -q -x -k "tcgen05 or draft or irope or golden or other_trees or max_ctx or bf16 or verify" 2>&1 | tail -2
for i in 1 2; do
  for v in new kv1s2; do
    lib=""; [ $v = kv1s2 ] && lib=tools/variants/kv1s2/libspecdec_b200.so
    for t in chain3 n8; do
      SDB_LIB=$lib timeout 300 python bench.py --tree $t --no-cpu-baseline --no-e2e --steps 30 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$v $t step', round(d['value'],1), 'attn', round(d['kernels_ms']['tree_attn']*1000,1), 'frac', round(d['roofline']['frac'],3))"
    done
    SDB_LIB=$lib timeout 300 python tools/draft_bench.py 2>&1 | tail -1 | cut -c1-200
  done
done
exit 0
