#!/bin/bash
# round-2 cycle 2: all GPU tests (incl. the benched-config parity and the
# reference suites through the shim), fixed-reference attention A/B, smoke, bench
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
T=gpurun_out/c2_times.txt
date +%T > $T
ab() {  # tag, lib, env...
  local tag=$1 lib=$2; shift 2
  env SDB_LIB=$lib "$@" timeout -s ABRT 120 python -X faulthandler tools/attn_bench.py c3 --iters 20 --reps 7 >> gpurun_out/c2_attn_$tag.jsonl 2>> gpurun_out/c2_attn.err
  echo "$tag $(date +%T)" >> $T
}
ab fix1 ""
ab fix0 tools/variants/fix0/libspecdec_b200.so
ab fix1 ""
ab fix0 tools/variants/fix0/libspecdec_b200.so
ab fix1_emu0 "" SDB_ATTN_EMU8=0
ab fix1_emu2 "" SDB_ATTN_EMU8=2
ab fix1_emu3 "" SDB_ATTN_EMU8=3
timeout -s ABRT 1500 python -X faulthandler -m pytest tests -m gpu -q -rf > gpurun_out/c2_pytest.txt 2>&1
echo "pytest $(date +%T)" >> $T
timeout -s ABRT 300 python -X faulthandler -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/c2_smoke.txt 2>&1
echo "smoke $(date +%T)" >> $T
timeout -s ABRT 400 python -X faulthandler bench.py > gpurun_out/c2_bench.json 2> gpurun_out/c2_bench.err
echo "bench $(date +%T)" >> $T
tail -3 gpurun_out/c2_pytest.txt
cat gpurun_out/c2_attn_*.jsonl
