#!/bin/bash
# stochastic acceptance evidence: new parity tests, bench c3 greedy/stochastic + c5, ncu of the c5 kernels
O=gpurun_out; T=${1:-st}; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_sampling.py tests/test_gpu_parity.py -q -m gpu -x > $O/${T}_pytest.txt 2>&1; tail -3 $O/${T}_pytest.txt
for c in "--config c3" "--config c3 --mode stochastic" "--config c5"; do
  timeout 600 python bench.py $c --no-cpu-baseline 2>>$O/${T}_bench.err | tee -a $O/${T}_bench.json
done
tail -5 $O/${T}_bench.err
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"row_stats|stochastic_walk|philox" -s 3 -c 3 -o $O/${T}_c5 \
  python bench.py --config c5 --steps 2 --warmup 3 --no-e2e --no-cpu-baseline > $O/${T}_ncu.log 2>&1; tail -1 $O/${T}_ncu.log
exit 0
