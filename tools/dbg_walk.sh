for v in "CUDA_LAUNCH_BLOCKING=1" "SDB_DIAG_SKIP_VALIDATE=1" "SDB_STOCH_EAGER=1" "A=1"; do
echo "== $v"; env SDB_WALK_CL=8 $v timeout 300 python bench.py --config c5 --steps 3 --warmup 3 --no-e2e --no-cpu-baseline 2>&1 | grep -o '"value": [0-9.]*\|Error.*\|line [0-9]*, in [a-z_]*' | head -8
done
