#!/bin/bash
# stochastic evidence after the walk rework: benches, launch list of the lazy C5 step, ncu of its kernels
O=gpurun_out; T=${1:-st9}; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_sampling.py tests/test_gpu_parity.py -q -m gpu -x > $O/${T}_pytest.txt 2>&1; tail -2 $O/${T}_pytest.txt
for c in "--config c5" "--config c3 --mode stochastic"; do
  timeout 600 python bench.py $c 2>>$O/${T}_bench.err | tee -a $O/${T}_bench.jsonl | cut -c 1-150
done
SDB_STOCH_EAGER=1 timeout 600 python bench.py --config c5 --no-cpu-baseline --no-e2e 2>>$O/${T}_bench.err | tee -a $O/${T}_bench_eager.jsonl | cut -c 1-120
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 60 --csv --log-file $O/${T}_launches.csv \
  python bench.py --config c5 --steps 2 --warmup 3 --no-e2e --no-cpu-baseline > $O/${T}_launch.log 2>&1; tail -1 $O/${T}_launch.log
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"row_stats|stochastic_walk|stochastic_validate" -s 3 -c 4 -o $O/${T}_c5 \
  python bench.py --config c5 --steps 1 --warmup 1 --no-e2e --no-cpu-baseline > $O/${T}_ncu.log 2>&1; tail -1 $O/${T}_ncu.log
exit 0
