# A/B of the SMs reserved for the concurrent greedy acceptance at C3 (same box, alternating)
for rep in 1 2; do
for r in 0 auto 12 16 20 24; do
  if [ "$r" = auto ]; then env_r=""; else env_r="SDB_RESERVE_SMS=$r"; fi
  echo "reserve=$r $(env $env_r python bench.py --config c3 --no-cpu-baseline --no-e2e --steps 30 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['value'],1), {k: round(v*1e3,1) for k,v in d['kernels_ms'].items()})")"
done
done
