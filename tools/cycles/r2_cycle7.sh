#!/bin/bash
# round-2 cycle 7 (restart baseline): all GPU tests, smoke, bench lines for every
# benched variant, the reference arm, a launch list of the default bench
cd $GRAFT_REPO_ROOT
O=gpurun_out; mkdir -p $O
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > $O/c7_smi.txt 2>&1
timeout -s ABRT 1500 python -X faulthandler -m pytest tests -m gpu -q -rf > $O/c7_pytest.txt 2>&1; tail -3 $O/c7_pytest.txt
timeout -s ABRT 300 python -X faulthandler -c "import __graft_entry__ as g; g.smoke()" > $O/c7_smoke.txt 2>&1; echo smoke rc=$?
for args in "" "--tree 65" "--tree chain3" "--tree n8" "--config c2" "--config c5" "--mode stochastic" "--config c4 --steps 10"; do
  echo "== $args" >> $O/c7_bench.jsonl
  timeout -s ABRT 400 python -X faulthandler bench.py $args --no-cpu-baseline >> $O/c7_bench.jsonl 2>> $O/c7_bench.err
done
timeout -s ABRT 600 python bench.py --impl reference --steps 3 --warmup 3 > $O/c7_ref.json 2> $O/c7_ref.err
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $O/c7_launches.csv \
  python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline > $O/c7_ncu_list.log 2>&1
exit 0
