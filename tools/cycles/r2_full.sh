#!/bin/bash
# round-2 full evidence pass: all GPU tests, smoke, default bench (with e2e + CPU baseline),
# the reference arm, bench lines of every config, launch list of the default bench
cd $GRAFT_REPO_ROOT
O=gpurun_out; mkdir -p $O
timeout -s ABRT 1800 python -X faulthandler -m pytest tests -m gpu -q -rf > $O/full_pytest.txt 2>&1; tail -3 $O/full_pytest.txt
timeout -s ABRT 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/full_smoke.txt 2>&1; echo smoke rc=$?; tail -2 $O/full_smoke.txt
timeout -s ABRT 600 python bench.py > $O/full_bench.json 2> $O/full_bench.err; echo bench rc=$?
timeout -s ABRT 900 python bench.py --impl reference > $O/full_ref.json 2> $O/full_ref.err; echo ref rc=$?
for args in "--tree 65" "--tree chain3" "--tree n8" "--config c2" "--config c5" "--mode stochastic" "--config c4 --steps 10"; do
  echo "== $args" >> $O/full_lines.jsonl
  timeout -s ABRT 400 python bench.py $args --no-cpu-baseline >> $O/full_lines.jsonl 2>> $O/full_lines.err
done
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $O/full_launches.csv python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline > /dev/null 2>&1
exit 0
