#!/bin/bash
# Full evidence pass on one B200: gpu parity tests, smoke, bench (N=1), the
# ncu launch list of the bench command, ncu --set full of the attention and
# acceptance kernels, reference arm.  Outputs under gpurun_out/<tag>_*.
# usage: bash tools/round_cycle.sh TAG [bench args...]
TAG=${1:-rc}; shift
O=gpurun_out; mkdir -p $O
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > $O/${TAG}_smi.txt 2>&1
nproc > $O/${TAG}_host.txt; lscpu | grep -E 'Model name|^CPU\(s\)' >> $O/${TAG}_host.txt
timeout 900 python -m pytest tests -q -m gpu -x > $O/${TAG}_pytest.txt 2>&1; tail -3 $O/${TAG}_pytest.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > $O/${TAG}_smoke.txt 2>&1; tail -2 $O/${TAG}_smoke.txt
timeout 600 python bench.py "$@" > $O/${TAG}_bench.json 2> $O/${TAG}_bench.err; cat $O/${TAG}_bench.json; tail -3 $O/${TAG}_bench.err
timeout 600 python bench.py --impl reference --steps 2 --warmup 1 > $O/${TAG}_ref.json 2>&1; tail -1 $O/${TAG}_ref.json
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $O/${TAG}_launches.csv \
  python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu-baseline "$@" > $O/${TAG}_launch.log 2>&1; tail -1 $O/${TAG}_launch.log
timeout 900 ncu --set full --clock-control none --import-source on -k regex:tree_attn_tcgen05 -s 1 -c 1 -o $O/${TAG}_attn \
  python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline "$@" > $O/${TAG}_ncu_attn.log 2>&1; tail -1 $O/${TAG}_ncu_attn.log
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"argmax_keys|row_stats|stochastic_walk|greedy_walk" -s 2 -c 2 -o $O/${TAG}_acc \
  python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline "$@" > $O/${TAG}_ncu_acc.log 2>&1; tail -1 $O/${TAG}_ncu_acc.log
exit 0
