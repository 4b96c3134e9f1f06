#!/bin/bash
# round-2: two-slot 1-CTA kernel -- all parity tests + sanitizers of the 1-CTA kernel
cd $GRAFT_REPO_ROOT
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_benched_configs.py tests/test_reference_suites_gpu.py -m gpu -q 2>&1 | tail -3
CS=/usr/local/cuda/bin/compute-sanitizer
for tool in memcheck synccheck racecheck; do
  echo "== $tool attn1"
  timeout 900 $CS --tool $tool --print-limit 5 python tools/sanitize_cases.py attn1 2>&1 | grep -E "SUMMARY|Error|error" | head -5
done
exit 0
