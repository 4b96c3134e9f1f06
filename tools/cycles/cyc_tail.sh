#!/bin/bash
# R = 65 tail row block: parity, then the attention time per tail cost weight
O=gpurun_out; T=${1:-tail}; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_parity.py -q -m gpu -x > $O/${T}_pytest.txt 2>&1; tail -2 $O/${T}_pytest.txt
for w in ${WS:-16 12 10 8 6}; do
  echo "== tail_w $w"
  SDB_ATTN_TAIL_W=$w timeout 600 python bench.py --tree 65 --no-cpu-baseline --no-e2e 2>>$O/${T}_bench.err | tee -a $O/${T}_bench.json | grep -o '"value": [0-9.]*\|"tree_attn": [0-9.]*'
done
echo "== R 64"; timeout 600 python bench.py --no-cpu-baseline --no-e2e 2>>$O/${T}_bench.err | grep -o '"value": [0-9.]*\|"tree_attn": [0-9.]*'
exit 0
