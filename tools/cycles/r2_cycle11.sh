#!/bin/bash
# round-2 cycle 11: warp-cooperative block-table cache in the TMA producers (+ 2 alternating
# softmax warpgroups) -- parity, A/B vs HEAD, exp2 emulation sweep, trace, bench lines
cd $GRAFT_REPO_ROOT
O=gpurun_out; mkdir -p $O
timeout -s ABRT 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_benched_configs.py -m gpu -q -x -k "tcgen05 or bench_step or draft or irope or golden or c4" > $O/c11_pytest.txt 2>&1; tail -3 $O/c11_pytest.txt
for rep in 1 2; do
  timeout -s ABRT 120 python tools/attn_bench.py c3 --iters 20 --reps 7 >> $O/c11_attn_new.jsonl 2>> $O/c11_attn.err
  SDB_LIB=tools/variants/old/libspecdec_b200.so timeout -s ABRT 120 python tools/attn_bench.py c3 --iters 20 --reps 7 >> $O/c11_attn_old.jsonl 2>> $O/c11_attn.err
done
for e in 0 2 3; do
  SDB_ATTN_EMU8=$e timeout -s ABRT 120 python tools/attn_bench.py c3 --iters 20 --reps 7 >> $O/c11_attn_emu$e.jsonl 2>> $O/c11_attn.err
done
for e in 1 2; do echo "== emu $e"; SDB_ATTN_EMU8=$e SDB_LIB=paper_2508_08192_b200/_lib/libspecdec_b200_trace.so timeout 120 python tools/trace_attn.py c3 2>&1 | grep -v "^[0-9]"; done > $O/c11_trace.txt
for args in "" "--tree 65" "--tree chain3" "--tree n8" "--config c2" "--config c4 --steps 10"; do
  echo "== $args" >> $O/c11_bench.jsonl
  timeout -s ABRT 400 python bench.py $args --no-cpu-baseline >> $O/c11_bench.jsonl 2>> $O/c11_bench.err
done
exit 0
