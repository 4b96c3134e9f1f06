"""Timeline of one pair-kernel worker on the fused R = 65 tail rows (trace
build with -DSDB_TRACE_WORKER=k): per item the MMA issuer's waits (V, P,
P^T of the previous item, tail reads) and the tail warps' S^T wait.
usage: SDB_LIB=tools/variants/<trace>/libspecdec_b200.so TRACE_TREE=65 python tools/trace_tail.py"""
import ctypes
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import bench  # noqa: E402
from paper_2508_08192_b200 import _lib  # noqa: E402
from paper_2508_08192_b200.attention import TreeVerifyAttention  # noqa: E402
from paper_2508_08192_b200.drafttree import tree_build  # noqa: E402
from paper_2508_08192_b200.sharding import shard_for  # noqa: E402

cfg = dict(bench.CONFIGS["c3"])
bench.TREE = bench.TREES[os.environ.get("TRACE_TREE", "65")]
lib = _lib.load()
dev = torch.device("cuda", 0)
shard = shard_for(0, 1, cfg["Hq"], cfg["Hkv"], cfg["V"])
x, R = bench.make_inputs(dict(cfg, V=1024), shard, dev)
mask, _, _, _ = tree_build(x.parent, x.n_rows, x.ctx_len)
attn = TreeVerifyAttention()
for _ in range(3):
    attn(x.q, x.k_pool, x.v_pool, x.block_table, x.ctx_len, x.tree_k, x.tree_v, mask, x.n_rows, cfg["d"] ** -0.5,
         max_ctx=cfg["ctx"], kernel=1)
torch.cuda.synchronize()
buf = np.zeros((24, 256), dtype=np.uint64)
fn = lib.sdb_debug_trace
fn.argtypes = [ctypes.c_void_p]
assert fn(buf.ctypes.data) == 0
ev = {"v_wait0": 18, "v_ok": 0, "p_ok": 1, "tp_ok": 21, "tread_ok": 22, "issued": 2, "sm_swait": 3, "sm_sok": 4,
      "sm_done": 5, "tail_sok": 23}
live = buf[1] > 0
t0 = int(buf[1][live].min())
print("item " + " ".join(f"{k:>9}" for k in ev))
for i in range(min(256, int(live.sum()) + 2)):
    row = []
    for k, e in ev.items():
        v = int(buf[e][i])
        row.append(f"{(v - t0) / 1000:9.1f}" if v else f"{'-':>9}")
    print(f"{i:4d} " + " ".join(row))
