make -C paper_2508_08192_b200/csrc trace -j8 > /dev/null 2>&1 || echo "trace build failed"
SDB_LIB=paper_2508_08192_b200/_lib/libspecdec_b200_trace.so python tools/trace_attn.py c3 2>&1 | tail -30
