#!/bin/bash
# round-2 cycle 5: tests + attention A/B + trace + bench lines (C3, R=65, C4) + ncu of the pair kernel
cd $GRAFT_REPO_ROOT
O=gpurun_out; mkdir -p $O
timeout -s ABRT 1500 python -X faulthandler -m pytest tests -m gpu -q -rf > $O/c5_pytest.txt 2>&1; tail -3 $O/c5_pytest.txt
for rep in 1 2; do
  timeout -s ABRT 120 python tools/attn_bench.py c3 --iters 20 --reps 7 >> $O/c5_attn_new.jsonl 2>> $O/c5_attn.err
  SDB_LIB=tools/variants/fix0/libspecdec_b200.so timeout -s ABRT 120 python tools/attn_bench.py c3 --iters 20 --reps 7 >> $O/c5_attn_fix0.jsonl 2>> $O/c5_attn.err
done
SDB_LIB=tools/variants/tr/libspecdec_b200.so timeout -s ABRT 120 python tools/trace_attn.py c3 > $O/c5_trace.txt 2>&1
for args in "" "--tree 65" "--config c4"; do
  echo "== $args" >> $O/c5_bench.jsonl
  timeout -s ABRT 400 python -X faulthandler bench.py $args >> $O/c5_bench.jsonl 2>> $O/c5_bench.err
done
timeout 900 ncu --set full --clock-control none --import-source on -k regex:tree_attn_tcgen05 -s 1 -c 1 -o $O/c5_attn \
  python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline > $O/c5_ncu_attn.log 2>&1; tail -1 $O/c5_ncu_attn.log
exit 0
