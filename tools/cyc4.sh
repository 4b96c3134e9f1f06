mkdir -p gpurun_out
timeout 600 python -m pytest tests -q -m gpu -x 2>&1 | tail -5
for e in 0 1 2 3 4; do SDB_ATTN_EMU8=$e timeout 120 python tools/attn_bench.py c3; done
SDB_LIB=paper_2508_08192_b200/_lib/libspecdec_b200_trace.so timeout 120 python tools/trace_attn.py c3 | tail -34
