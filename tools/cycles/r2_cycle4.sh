#!/bin/bash
# round-2 cycle 4: K/V ring depth A/B under the fixed-reference softmax,
# synccheck / racecheck of the pair kernel (o_last), bench lines
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
ab() {  # tag, lib, env...
  local tag=$1 lib=$2; shift 2
  env SDB_LIB=$lib "$@" timeout -s ABRT 120 python -X faulthandler tools/attn_bench.py c3 --iters 20 --reps 7 >> gpurun_out/c4_attn_$tag.jsonl 2>> gpurun_out/c4_attn.err
}
for rep in 1 2; do
  ab k6v3 ""
  for v in k6v4 k5v4 k5v5; do ab $v tools/variants/$v/libspecdec_b200.so; done
done
CS=/usr/local/cuda/bin/compute-sanitizer
for tool in synccheck racecheck; do
  echo "== $tool attn" >> gpurun_out/c4_sanitize.txt
  timeout -s ABRT 600 $CS --tool $tool --print-limit 5 python tools/sanitize_cases.py attn >> gpurun_out/c4_sanitize.txt 2>&1
  echo "rc=$?" >> gpurun_out/c4_sanitize.txt
done
for args in "" "--tree chain3" "--tree n8" "--tree 65" "--config c2" "--config c5" "--mode stochastic"; do
  echo "== $args" >> gpurun_out/c4_bench.jsonl
  timeout -s ABRT 400 python -X faulthandler bench.py $args >> gpurun_out/c4_bench.jsonl 2>> gpurun_out/c4_bench.err
done
grep -E "==|SUMMARY|rc=" gpurun_out/c4_sanitize.txt
for f in gpurun_out/c4_attn_*.jsonl; do echo $f; cut -c1-120 $f; done
