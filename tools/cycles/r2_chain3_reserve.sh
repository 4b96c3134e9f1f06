#!/bin/bash
# round-2: SMs reserved for the concurrent scan at the HBM-bound small trees
cd $GRAFT_REPO_ROOT
for t in chain3 n8; do
  for k in 0 8 12 16 20; do
    if [ $k = 0 ]; then env=""; else env="SDB_RESERVE_SMS=$k"; fi
    env $env timeout 300 python bench.py --tree $t --no-cpu-baseline --no-e2e --steps 30 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$t reserve ${k:-auto}', round(d['value'],1))"
  done
done
exit 0
