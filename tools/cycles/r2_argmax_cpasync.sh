#!/bin/bash
# round-2: greedy scan through a per-thread cp.async ring (6 / 4 stages vs plain loads), reserve sweep
cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_benched_configs.py tests/test_gpu_sampling.py -m gpu -q -x -k "greedy or argmax or bench_step or golden or fsm or shard" 2>&1 | tail -2
for i in 1 2; do
  for v in s6 am4 am0; do
    lib=""; [ $v != s6 ] && lib=tools/variants/$v/libspecdec_b200.so
    SDB_LIB=$lib timeout 300 python bench.py --no-cpu-baseline --no-e2e --steps 30 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$v c3 step', round(d['value'],1), 'accept alone', round(d['kernels_ms']['accept']*1000,1), 'attn', round(d['kernels_ms']['tree_attn']*1000,1))"
  done
done
for k in 12 14 16 18 20; do
  SDB_RESERVE_SMS=$k timeout 300 python bench.py --no-cpu-baseline --no-e2e --steps 30 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('s6 reserve $k step', round(d['value'],1))"
done
timeout 600 python bench.py --steps 20 > gpurun_out/cp_bench_default.json 2> gpurun_out/cp_bench_default.err; echo "default bench rc=$?"; python -c "import json; d=json.load(open('gpurun_out/cp_bench_default.json')); print(d['value'], d['cpu_baseline']['kind'], d['cpu_baseline']['value'], d['cpu_baseline']['sample'][:100])"
exit 0
