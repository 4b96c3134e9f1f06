#!/bin/bash
# round-2 final profiles: ncu --set full of the 1-CTA kernel at chain-3 (two S slots, 3-stage ring)
cd $GRAFT_REPO_ROOT
O=gpurun_out; mkdir -p $O
B="python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline"
timeout 600 ncu --set full --clock-control none --import-source on -k regex:tree_attn_tcgen05_kernel -s 2 -c 1 -o $O/r2p2_chain3 $B --tree chain3 > $O/r2p2_chain3.log 2>&1; tail -1 $O/r2p2_chain3.log
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 200 --csv --log-file $O/r2p2_chain3_launches.csv $B --tree chain3 > /dev/null 2>&1
exit 0
