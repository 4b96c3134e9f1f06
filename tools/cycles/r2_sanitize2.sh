#!/bin/bash
# round-2: re-check after the o_done (1-CTA) and tmem_base (pair) changes
cd $GRAFT_REPO_ROOT
O=gpurun_out; mkdir -p $O
CS=/usr/local/cuda/bin/compute-sanitizer
for c in "racecheck attn" "synccheck attn1" "memcheck attn1" "synccheck attn" ; do
  set -- $c
  echo "== $1 $2" >> $O/r2_sanitize2.txt
  timeout -s ABRT 900 $CS --tool $1 --print-limit 10 python tools/sanitize_cases.py $2 >> $O/r2_sanitize2.txt 2>&1
  echo "rc=$?" >> $O/r2_sanitize2.txt
done
grep -E "^==|SUMMARY|rc=|Error|error" $O/r2_sanitize2.txt | head -40
timeout -s ABRT 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_benched_configs.py -m gpu -q -x > $O/r2_san2_pytest.txt 2>&1; tail -2 $O/r2_san2_pytest.txt
for args in "--tree chain3" "--tree n8" ""; do timeout 300 python bench.py $args --no-cpu-baseline --no-e2e --steps 20 | cut -c1-300; done
exit 0
