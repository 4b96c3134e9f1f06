mkdir -p gpurun_out
timeout 600 python -m pytest tests -q -m gpu -x > gpurun_out/pytest_c6.txt 2>&1; tail -2 gpurun_out/pytest_c6.txt
timeout 300 python bench.py > gpurun_out/bench_c6.txt 2> gpurun_out/bench_c6.err; cat gpurun_out/bench_c6.txt; tail -3 gpurun_out/bench_c6.err
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -s 40 -c 40 --csv --log-file gpurun_out/launches_c6.csv python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline > /dev/null 2>&1
timeout 500 ncu --set full --clock-control none --import-source on -k regex:tree_attn_tcgen05 -s 1 -c 1 -o gpurun_out/prof_c6 python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline > /dev/null 2>&1
timeout 500 ncu --set full --clock-control none --import-source on -k regex:argmax_keys -s 1 -c 1 -o gpurun_out/prof_c6_accept python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline > /dev/null 2>&1
ls gpurun_out
