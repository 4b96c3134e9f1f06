mkdir -p gpurun_out
timeout 600 python -m pytest tests -q -m gpu -x 2>&1 | tail -5
for cg in 1 2; do for e in 0 1 2; do SDB_ATTN_CTA_GROUP=$cg SDB_ATTN_EMU=$e timeout 120 python tools/attn_bench.py c3; done; done
SDB_LIB=paper_2508_08192_b200/_lib/libspecdec_b200_trace.so timeout 120 python tools/trace_attn.py c3 | tail -32
