#!/bin/bash
O=gpurun_out; T=${1:-sh}; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_sampling.py -q -m gpu -x > $O/${T}_pytest.txt 2>&1; tail -15 $O/${T}_pytest.txt
SDB_BENCH_BACKEND=gloo timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29533 bench.py --gpus 2 --config c5 --steps 3 --warmup 3 --no-e2e > $O/${T}_gloo_c5.txt 2>&1; tail -3 $O/${T}_gloo_c5.txt | cut -c1-600
exit 0
