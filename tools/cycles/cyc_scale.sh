#!/bin/bash
O=gpurun_out; T=${1:-sc}; mkdir -p $O
for c in "--config c2" "--config c4"; do
  timeout 900 python bench.py $c --no-cpu-baseline --no-e2e --steps 20 2>>$O/${T}_bench.err | tee -a $O/${T}_bench.json | cut -c 1-160
  grep -o '"kernels_ms": {[^}]*}' $O/${T}_bench.json | tail -1; grep -o '"roofline": {[^}]*}' $O/${T}_bench.json | tail -1
done
for g in 1 2 4 8; do timeout 600 python tools/attn_bench.py c3 --gpus $g >> $O/${T}_attn.jsonl 2>&1; done
for g in 1 8; do timeout 600 python tools/attn_bench.py c4 --gpus $g >> $O/${T}_attn.jsonl 2>&1; done
timeout 600 python tools/attn_bench.py c2 >> $O/${T}_attn.jsonl 2>&1
cat $O/${T}_attn.jsonl; tail -3 $O/${T}_bench.err
exit 0
