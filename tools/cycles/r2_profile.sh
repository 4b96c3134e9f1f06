#!/bin/bash
# round-2 profiles of the final kernels: ncu --set full of the pair attention
# (C3 bench step), the greedy scan, the 1-CTA kernel at chain-3; DRAM bytes of
# the C5 lazy chain; launch lists of the C3 / C5 bench commands
cd $GRAFT_REPO_ROOT
O=gpurun_out; mkdir -p $O
B="python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:tree_attn_tcgen05_pair -s 2 -c 1 -o $O/r2p_attn $B > $O/r2p_attn.log 2>&1; tail -1 $O/r2p_attn.log
timeout 600 ncu --set full --clock-control none -k regex:argmax_keys -s 2 -c 1 -o $O/r2p_argmax $B > $O/r2p_argmax.log 2>&1; tail -1 $O/r2p_argmax.log
timeout 600 ncu --set full --clock-control none -k regex:tree_attn_tcgen05_kernel -s 2 -c 1 -o $O/r2p_chain3 $B --tree chain3 > $O/r2p_chain3.log 2>&1; tail -1 $O/r2p_chain3.log
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:"row_stats|stochastic_walk|stochastic_validate|philox|lazy_walk" -c 80 --csv --log-file $O/r2p_c5_dram.csv $B --config c5 > $O/r2p_c5.log 2>&1; tail -1 $O/r2p_c5.log
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $O/r2p_c3_launches.csv $B > $O/r2p_c3_list.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $O/r2p_c5_launches.csv $B --config c5 > $O/r2p_c5_list.log 2>&1
ls -la $O/r2p_*
exit 0
