#!/bin/bash
# re-entry check: all GPU tests, smoke, default bench line
cd $GRAFT_REPO_ROOT
O=gpurun_out; mkdir -p $O
timeout -s ABRT 1800 python -X faulthandler -m pytest tests -m gpu -q -rf > $O/re_pytest.txt 2>&1; tail -3 $O/re_pytest.txt
timeout -s ABRT 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/re_smoke.txt 2>&1; echo smoke rc=$?; tail -2 $O/re_smoke.txt
timeout -s ABRT 600 python bench.py > $O/re_bench.json 2> $O/re_bench.err; echo bench rc=$?; cut -c1-600 $O/re_bench.json
exit 0
