#!/bin/bash
# C2 (bs 1) pair-kernel phase trace (worker 0 + every worker's start / end)
cd $GRAFT_REPO_ROOT
SDB_LIB=paper_2508_08192_b200/_lib/libspecdec_b200_trace.so timeout 300 python tools/trace_attn.py c2 2>&1 | tail -45
exit 0
