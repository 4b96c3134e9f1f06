#!/bin/bash
# round-2 cycle 12: attention time model with the K/V stream (HBM-bound small trees: no SM reserve,
# scan after the attention) -- bench lines chain3 / n8 / c3, parity tests
cd $GRAFT_REPO_ROOT
O=gpurun_out; mkdir -p $O
for args in "--tree chain3" "--tree n8" "" "--tree chain3 --kernel 2"; do
  echo "== $args" >> $O/c12_bench.jsonl
  timeout -s ABRT 400 python bench.py $args --no-cpu-baseline >> $O/c12_bench.jsonl 2>> $O/c12_bench.err
done
timeout -s ABRT 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_benched_configs.py -m gpu -q -x > $O/c12_pytest.txt 2>&1; tail -3 $O/c12_pytest.txt
exit 0
