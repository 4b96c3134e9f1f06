#!/bin/bash
# round-2: default bench line (stock-reference cpu_baseline from spawned workers) and the 2-rank gloo path
cd $GRAFT_REPO_ROOT
s=$(date +%s); timeout 900 python bench.py > gpurun_out/bc_default.json 2> gpurun_out/bc_default.err; echo "default rc=$? wall $(( $(date +%s) - s )) s"
python -c "import json; d=json.load(open('gpurun_out/bc_default.json')); print(d['value'], d['e2e']['value'], d['cpu_baseline']['kind'], d['cpu_baseline']['value'], d['cpu_baseline']['cores'], d['parity']['ok'])"
SDB_BENCH_BACKEND=gloo timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29531 bench.py --gpus 2 --steps 5 --warmup 3 --no-e2e 2>&1 | tail -2 | cut -c1-400
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29532 bench.py --impl reference --gpus 2 --steps 2 --warmup 1 2>&1 | tail -1 | cut -c1-300
exit 0
