#!/bin/bash
# round-2 cycle 3: clock64 traces of the pair kernel (fixed reference vs
# running max, exp2 emulation 0 / 1), sanitizers on the pair kernel and the
# stochastic cluster walk
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
for v in tr_fix1 tr_fix0; do
  for emu in 0 1; do
    echo "== $v emu $emu" >> gpurun_out/c3_trace.txt
    SDB_LIB=tools/variants/$v/libspecdec_b200.so SDB_ATTN_EMU8=$emu timeout -s ABRT 120 python tools/trace_attn.py c3 >> gpurun_out/c3_trace.txt 2>&1
  done
done
CS=/usr/local/cuda/bin/compute-sanitizer
for tool in racecheck synccheck memcheck; do
  for c in attn stoch; do
    echo "== $tool $c" >> gpurun_out/c3_sanitize.txt
    timeout -s ABRT 600 $CS --tool $tool --print-limit 20 python tools/sanitize_cases.py $c >> gpurun_out/c3_sanitize.txt 2>&1
    echo "rc=$?" >> gpurun_out/c3_sanitize.txt
  done
done
grep -E "==|ERROR SUMMARY|rc=|ok" gpurun_out/c3_sanitize.txt
