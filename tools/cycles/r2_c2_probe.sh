#!/bin/bash
# C2 (bs 1) latency structure: attention device time vs context and worker count; launch list of the c2 bench
cd $GRAFT_REPO_ROOT
O=gpurun_out; mkdir -p $O
timeout 300 python tools/c2_probe.py 128,1024,8192 0,8,16,32,48,64,74 > $O/c2p_probe.jsonl 2>&1; cat $O/c2p_probe.jsonl | tr '\n' ' '; echo
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 60 --csv --log-file $O/c2p_launches.csv python bench.py --config c2 --steps 2 --warmup 3 --no-e2e --no-cpu-baseline > /dev/null 2>&1
python tools/launch_summary.py $O/c2p_launches.csv 2>/dev/null | tail -15
exit 0
