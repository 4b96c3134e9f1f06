#!/bin/bash
# One GPU iteration: parity tests, bench, optional ncu capture of the attention kernel.
# usage: bash tools/gpu_cycle.sh [tag] [test-filter] [ncu:0|1] [bench args...]
TAG=${1:-run}; FILT=${2:-}; NCU=${3:-1}; shift 3 2>/dev/null
mkdir -p gpurun_out
if [ -n "$FILT" ]; then K="-k"; else K=""; fi
timeout 600 python -m pytest tests -q -m gpu -x ${K:+$K "$FILT"} > gpurun_out/pytest_$TAG.txt 2>&1; tail -3 gpurun_out/pytest_$TAG.txt
timeout 600 python bench.py "$@" > gpurun_out/bench_$TAG.txt 2> gpurun_out/bench_$TAG.err; cat gpurun_out/bench_$TAG.txt; tail -3 gpurun_out/bench_$TAG.err
if [ "$NCU" = "1" ]; then
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:tree_attn_tcgen05 -s 1 -c 1 -o gpurun_out/prof_$TAG python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline "$@" > gpurun_out/ncu_$TAG.log 2>&1; tail -1 gpurun_out/ncu_$TAG.log
fi
