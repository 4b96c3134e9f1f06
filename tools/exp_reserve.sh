# A/B of the SMs reserved for the concurrent greedy acceptance at C3 (same box, alternating)
for rep in 1 2; do
for r in auto 20 22 23 24; do
  if [ "$r" = auto ]; then env_r=""; else env_r="SDB_RESERVE_SMS=$r"; fi
  echo "reserve=$r $(env $env_r python bench.py --config c3 --no-cpu-baseline --no-e2e --steps 30 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['value'],1), round(d['kernels_ms']['tree_attn']*1e3,1), d['clocks']['sm_mhz'])")"
done
done
