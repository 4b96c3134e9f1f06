timeout 600 python -m pytest tests -q -m gpu -x 2>&1 | tail -2
for e in 0 1 2 3 4; do SDB_ATTN_EMU8=$e timeout 120 python tools/attn_bench.py c3; done
