#!/bin/bash
# round-2: sanitizers after the 2-CTA row split (stoch) and the two-slot 1-CTA kernel (attn1)
cd $GRAFT_REPO_ROOT
O=gpurun_out; mkdir -p $O
CS=/usr/local/cuda/bin/compute-sanitizer
for c in "memcheck stoch" "synccheck stoch" "racecheck stoch" "memcheck attn1" "synccheck attn1" "racecheck attn1"; do
  set -- $c
  echo "== $1 $2" >> $O/r2_sanitize3.txt
  timeout -s ABRT 900 $CS --tool $1 --print-limit 10 python tools/sanitize_cases.py $2 >> $O/r2_sanitize3.txt 2>&1
  echo "rc=$?" >> $O/r2_sanitize3.txt
done
grep -E "^==|SUMMARY|rc=" $O/r2_sanitize3.txt
exit 0
