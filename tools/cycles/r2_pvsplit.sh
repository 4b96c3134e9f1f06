#!/bin/bash
# split-PV handshake A/B: attention parity tests on the new build, then
# interleaved attention-alone and bench-step timings, new vs -DSDB_PV_SPLIT=0
cd $GRAFT_REPO_ROOT
O=gpurun_out; mkdir -p $O
timeout -s ABRT 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_benched_configs.py -m gpu -q -k "tcgen05 or verifier or draft or fused or c3 or c4 or irope" > $O/pv_pytest.txt 2>&1; tail -3 $O/pv_pytest.txt
NS=tools/variants/nosplit/libspecdec_b200.so
for i in 1 2 3; do
  echo "split   $(timeout 300 python tools/attn_bench.py c3 | cut -c1-120)"
  echo "nosplit $(SDB_LIB=$NS timeout 300 python tools/attn_bench.py c3 | cut -c1-120)"
done
for i in 1 2; do
  echo "split   step $(timeout 300 python bench.py --no-e2e --no-cpu-baseline | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(d["value"], d["kernels_ms"], d["parity"]["ok"])')"
  echo "nosplit step $(SDB_LIB=$NS timeout 300 python bench.py --no-e2e --no-cpu-baseline | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(d["value"], d["kernels_ms"], d["parity"]["ok"])')"
done
echo "split c4 $(timeout 300 python tools/attn_bench.py c4 --iters 5 --reps 3 | cut -c1-120)"
echo "nosplit c4 $(SDB_LIB=$NS timeout 300 python tools/attn_bench.py c4 --iters 5 --reps 3 | cut -c1-120)"
exit 0
