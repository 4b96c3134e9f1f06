#!/bin/bash
# round-2 cycle 9: two warpgroups alternating items -- parity, A/B vs the
# previous 3-warpgroup kernel, exp2 emulation sweep, phase trace, bench line
cd $GRAFT_REPO_ROOT
O=gpurun_out; mkdir -p $O
timeout -s ABRT 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_benched_configs.py -m gpu -q -x -k "tcgen05 or bench_step or draft or irope or golden or c4" > $O/c9_pytest.txt 2>&1; tail -3 $O/c9_pytest.txt
for rep in 1 2; do
  timeout -s ABRT 120 python tools/attn_bench.py c3 --iters 20 --reps 7 >> $O/c9_attn_new.jsonl 2>> $O/c9_attn.err
  SDB_LIB=tools/variants/old/libspecdec_b200.so timeout -s ABRT 120 python tools/attn_bench.py c3 --iters 20 --reps 7 >> $O/c9_attn_old.jsonl 2>> $O/c9_attn.err
done
for e in 0 2 3 4; do
  SDB_ATTN_EMU8=$e timeout -s ABRT 120 python tools/attn_bench.py c3 --iters 20 --reps 7 >> $O/c9_attn_emu$e.jsonl 2>> $O/c9_attn.err
done
SDB_LIB=paper_2508_08192_b200/_lib/libspecdec_b200_trace.so timeout -s ABRT 120 python tools/trace_attn.py c3 > $O/c9_trace.txt 2>&1
for args in "" "--tree 65" "--config c4 --steps 10"; do
  echo "== $args" >> $O/c9_bench.jsonl
  timeout -s ABRT 400 python bench.py $args --no-cpu-baseline >> $O/c9_bench.jsonl 2>> $O/c9_bench.err
done
exit 0
