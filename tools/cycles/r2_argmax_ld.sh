cd $GRAFT_REPO_ROOT
for v in "" tools/variants/ld1/libspecdec_b200.so tools/variants/ld2/libspecdec_b200.so; do
  echo "== lib $v"
  SDB_LIB=$v timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,lts__t_sectors_srcunit_tex_op_read.sum --clock-control none -k regex:argmax_keys -s 3 -c 2 python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline 2>&1 | grep -E "argmax|duration|bytes_read|sectors" | head -8
  SDB_LIB=$v timeout 300 python bench.py --steps 20 --no-e2e --no-cpu-baseline | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('step', round(d['value'],1), 'accept', round(d['kernels_ms']['accept']*1000,1))"
done
