#!/bin/bash
cd $GRAFT_REPO_ROOT
O=gpurun_out; mkdir -p $O
./tools/micro/mufu_bench > $O/c6_mufu.txt 2>&1
./tools/micro/mma_bench > $O/c6_mma.txt 2>&1
timeout -s ABRT 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_benched_configs.py -m gpu -q -x -k "tcgen05 or bench_step or draft or irope or golden" > $O/c6_pytest.txt 2>&1; tail -3 $O/c6_pytest.txt
for rep in 1 2; do
  timeout -s ABRT 120 python tools/attn_bench.py c3 --iters 20 --reps 7 >> $O/c6_attn_new.jsonl 2>> $O/c6_attn.err
  SDB_LIB=tools/variants/fix0/libspecdec_b200.so timeout -s ABRT 120 python tools/attn_bench.py c3 --iters 20 --reps 7 >> $O/c6_attn_fix0.jsonl 2>> $O/c6_attn.err
done
SDB_ATTN_EMU8=1 timeout -s ABRT 120 python tools/attn_bench.py c3 --iters 20 --reps 7 >> $O/c6_attn_emu1.jsonl 2>> $O/c6_attn.err
SDB_LIB=tools/variants/tr/libspecdec_b200.so timeout -s ABRT 120 python tools/trace_attn.py c3 > $O/c6_trace.txt 2>&1
exit 0
