#!/bin/bash
# round-2: trace of a fused-tail worker (R = 65, worker 40 of 74 runs last-block units)
cd $GRAFT_REPO_ROOT
SDB_LIB=tools/variants/trace40/libspecdec_b200.so TRACE_TREE=65 timeout 300 python tools/trace_tail.py 2>&1 | head -150
exit 0
