set -x
mkdir -p gpurun_out
timeout 900 python -m pytest tests -q -m gpu -x > gpurun_out/pytest_c1.txt 2>&1; tail -3 gpurun_out/pytest_c1.txt
for cg in 1 2; do for e in 0 1 2; do SDB_ATTN_CTA_GROUP=$cg SDB_ATTN_EMU=$e timeout 120 python tools/attn_bench.py c3; done; done
timeout 300 python bench.py > gpurun_out/bench_c1.txt 2> gpurun_out/bench_c1.err; cat gpurun_out/bench_c1.txt; tail -3 gpurun_out/bench_c1.err
timeout 600 ncu --set full --clock-control none --import-source on -k regex:tree_attn_tcgen05 -s 1 -c 1 -o gpurun_out/prof_c1 python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/ncu_c1.log 2>&1; tail -2 gpurun_out/ncu_c1.log
