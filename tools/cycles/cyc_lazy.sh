#!/bin/bash
# lazy vs eager stochastic acceptance: parity, c5/c3 benches both ways (+ walk cluster sizes), launch list of the lazy chain
O=gpurun_out; T=${1:-lz}; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_sampling.py tests/test_gpu_parity.py -q -m gpu -x > $O/${T}_pytest.txt 2>&1; tail -3 $O/${T}_pytest.txt
run() { echo "== $*"; env "$@" timeout 600 python bench.py $C --no-cpu-baseline --no-e2e 2>>$O/${T}_bench.err | tee -a $O/${T}_bench.json | grep -o '"value": [0-9.]*\|"kernels_ms": {[^}]*}'; }
C="--config c5"; run A=1; run SDB_STOCH_EAGER=1; run SDB_WALK_CL=8; run SDB_WALK_CL=4
C="--config c3 --mode stochastic"; run A=1; run SDB_STOCH_EAGER=1
tail -3 $O/${T}_bench.err
for cl in 4 8; do
SDB_WALK_CL=$cl SDB_DIAG_SKIP_VALIDATE=1 timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"row_stats|stochastic_walk|lazy|philox" -c 14 --csv --log-file $O/${T}_cl$cl.csv python bench.py --config c5 --steps 1 --warmup 3 --no-e2e --no-cpu-baseline > /dev/null 2>&1
done
exit 0
