#!/bin/bash
# round-2: compute-sanitizer memcheck / racecheck / synccheck of the final
# pair kernel, the 1-CTA kernel, the stochastic cluster walk (+ row stats, validation)
cd $GRAFT_REPO_ROOT
O=gpurun_out; mkdir -p $O
CS=/usr/local/cuda/bin/compute-sanitizer
for case in attn attn1 stoch; do
  for tool in memcheck synccheck racecheck; do
    echo "== $tool $case" >> $O/r2_sanitize.txt
    timeout -s ABRT 900 $CS --tool $tool --print-limit 10 python tools/sanitize_cases.py $case >> $O/r2_sanitize.txt 2>&1
    echo "rc=$?" >> $O/r2_sanitize.txt
  done
done
grep -E "^==|SUMMARY|rc=" $O/r2_sanitize.txt
exit 0
