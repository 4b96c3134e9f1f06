#!/bin/bash
# round-2 cycle 1: GPU tests on the new code + attention register-split A/B
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > gpurun_out/c1_smi.txt
for v in r0 r32 default; do
  if [ $v = default ]; then lib=""; else lib=tools/variants/$v/libspecdec_b200.so; fi
  for rep in 1 2; do
    SDB_LIB=$lib timeout 300 python tools/attn_bench.py c3 --iters 20 --reps 7 >> gpurun_out/c1_attn_$v.jsonl 2>> gpurun_out/c1_attn.err
  done
done
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/c1_pytest.txt 2>&1
timeout 300 python bench.py > gpurun_out/c1_bench.json 2> gpurun_out/c1_bench.err
tail -3 gpurun_out/c1_pytest.txt
cat gpurun_out/c1_attn_*.jsonl
