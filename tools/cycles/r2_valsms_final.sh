#!/bin/bash
# persistent validation scan as the default: all GPU tests, C5 / C3-stochastic lines, C5 launch list,
# ncu full of the persistent scan kernel, memcheck of one C5 step
cd $GRAFT_REPO_ROOT
O=gpurun_out; mkdir -p $O
timeout -s ABRT 1800 python -X faulthandler -m pytest tests -m gpu -q -rf > $O/vf_pytest.txt 2>&1; tail -3 $O/vf_pytest.txt
for args in "--config c5" "--mode stochastic"; do
  timeout 400 python bench.py $args --no-cpu-baseline >> $O/vf_lines.jsonl 2>> $O/vf_lines.err
  tail -1 $O/vf_lines.jsonl | cut -c1-300
done
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 200 --csv --log-file $O/vf_c5_launches.csv python bench.py --config c5 --steps 2 --warmup 3 --no-e2e --no-cpu-baseline > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:stochastic_validate_persistent -c 1 -o $O/vf_validate python bench.py --config c5 --steps 1 --warmup 3 --no-e2e --no-cpu-baseline > $O/vf_ncu.log 2>&1; echo ncu rc=$?
timeout 600 compute-sanitizer --tool memcheck --kernel-name regex:stochastic_validate_persistent python bench.py --config c5 --steps 1 --warmup 3 --no-e2e --no-cpu-baseline > $O/vf_memcheck.txt 2>&1; echo memcheck rc=$?; grep -E "ERROR SUMMARY" $O/vf_memcheck.txt | tail -1
exit 0
