timeout 600 python -m pytest tests -q -m gpu -x 2>&1 | tail -2
timeout 300 python bench.py --no-cpu-baseline --no-e2e 2>&1 | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(d['value'], d['kernels_ms'], d['roofline']['accept_hbm_frac'])"
