#!/bin/bash
# round-2 final evidence pass (after the persistent validation scan): all GPU tests, smoke, default bench
# (e2e + stock-reference CPU baseline), the reference arm, every config line, launch lists of C3 and C5
cd $GRAFT_REPO_ROOT
O=gpurun_out; mkdir -p $O
timeout -s ABRT 1800 python -X faulthandler -m pytest tests -m gpu -q -rf > $O/f4_pytest.txt 2>&1; tail -3 $O/f4_pytest.txt
timeout -s ABRT 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/f4_smoke.txt 2>&1; echo smoke rc=$?; tail -2 $O/f4_smoke.txt
timeout -s ABRT 600 python bench.py > $O/f4_bench.json 2> $O/f4_bench.err; echo bench rc=$?; cut -c1-200 $O/f4_bench.json
timeout -s ABRT 900 python bench.py --impl reference > $O/f4_ref.json 2> $O/f4_ref.err; echo ref rc=$?; cut -c1-200 $O/f4_ref.json
rm -f $O/f4_lines.jsonl
for args in "--tree 65" "--tree chain3" "--tree n8" "--config c2" "--config c5" "--mode stochastic" "--config c4 --steps 10"; do
  echo "== $args" >> $O/f4_lines.jsonl
  timeout -s ABRT 400 python bench.py $args --no-cpu-baseline >> $O/f4_lines.jsonl 2>> $O/f4_lines.err
done
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"sdb|tree_|argmax|walk|compact|fixup|clear" -c 400 --csv --log-file $O/f4_c3_launches.csv python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline > /dev/null 2>&1; echo c3 launches rc=$?
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum --clock-control none -k regex:"sdb|row_stats|stochastic|philox|walk|clear" -c 400 --csv --log-file $O/f4_c5_launches.csv python bench.py --config c5 --steps 2 --warmup 3 --no-e2e --no-cpu-baseline > /dev/null 2>&1; echo c5 launches rc=$?
timeout 900 ncu --set full --clock-control none --import-source on -k regex:stochastic_validate_persistent -c 1 -o $O/f4_validate python bench.py --config c5 --steps 1 --warmup 3 --no-e2e --no-cpu-baseline > /dev/null 2>&1; echo ncu validate rc=$?
exit 0
