"""Phase timeline of row_stats_kernel (target row of sequence 0, every launch)
from the SDB_TRACE build: SDB_LIB=paper_2508_08192_b200/_lib/libspecdec_b200_trace.so
python tools/trace_rowstats.py [lazy|eager]"""
import ctypes
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import bench  # noqa: E402
from paper_2508_08192_b200 import _lib  # noqa: E402
from paper_2508_08192_b200.sampling import StochasticAcceptor  # noqa: E402
from paper_2508_08192_b200.sharding import shard_for  # noqa: E402

cfg = bench.CONFIGS["c5"]
lib = _lib.load()
dev = torch.device("cuda", 0)
x, R = bench.make_inputs(cfg, shard_for(0, 1, cfg["Hq"], cfg["Hkv"], cfg["V"]), dev, mode="stochastic")
lazy = (sys.argv[1] if len(sys.argv) > 1 else "lazy") == "lazy"
acc = StochasticAcceptor(lazy=lazy, levels=bench._tree_levels(tuple(bench._augment(bench.TREE))))
for _ in range(2):
    res = acc(x.logits, x.draft_logits, 1.0, 0.9, x.parent, x.n_rows, x.tokens, seeds=x.seeds, steps=x.steps)
torch.cuda.synchronize()
buf = np.zeros((16, 8), dtype=np.uint64)
cnt = np.zeros(1, dtype=np.uint32)
fn = lib.sdb_debug_st_trace
fn.argtypes = [ctypes.c_void_p, ctypes.c_void_p]
assert fn(buf.ctypes.data, cnt.ctypes.data) == 0
names = ["max pass", "normaliser+hist", "window", "mass above+collect", "exact cut", "-", "-"]
print("launches", int(cnt[0]))
for i in range(16):
    if not buf[i, 0]:
        continue
    t = buf[i].astype(np.int64)
    d = [int(t[k + 1] - t[k]) if t[k + 1] and t[k] else None for k in range(5)]
    print(i, " ".join(f"{names[k]}={d[k]}" for k in range(5)))
