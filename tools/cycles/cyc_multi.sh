# multi-rank paths on one GPU (gloo; NCCL on a multi-GPU box runs the same calls)
for c in "--config c3" "--config c3 --mode stochastic" "--config c5"; do
SDB_BENCH_BACKEND=gloo timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29541 bench.py --gpus 2 $c --steps 3 --warmup 3 --no-e2e 2>&1 | grep -E '^\{' | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['config']['workload'], d['n_gpus'], round(d['value'],1), d['config']['graph'], d['mean_accepted'])"
done
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29542 bench.py --impl reference --gpus 2 --steps 1 --warmup 1 2>&1 | grep -E '^\{' | cut -c1-200
