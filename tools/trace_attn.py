"""Phase timeline of the pair attention kernel (worker 0) from the debug
build: SDB_LIB=paper_2508_08192_b200/_lib/libspecdec_b200_trace.so
python tools/trace_attn.py [config]"""
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

cfg = bench.CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "c3"]
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
buf = np.zeros((16, 256), dtype=np.uint64)
fn = lib.sdb_debug_trace
fn.argtypes = [ctypes.c_void_p]
assert fn(buf.ctypes.data) == 0
t0 = buf[buf > 0].min()
b = buf.astype(np.int64) - int(t0)
names = ["mma_pwait0", "mma_pok0", "mma_issued0", "mma_pwait1", "mma_pok1", "mma_issued1",
         "sm0_swait", "sm0_sok", "sm0_done", "sm1_swait", "sm1_sok", "sm1_done", "mma_vwait", "mma_vok"]
n = int((buf[7] > 0).sum())
print("iterations traced", n)
for it in range(min(n, 40)):
    row = " ".join(f"{names[e][:9]}={b[e, it]:>8d}" for e in (12, 13, 0, 1, 2, 3, 4, 5, 6, 7, 8, 9, 10, 11))
    print(it, row)
it = np.arange(5, min(n, 60))
per_it = np.diff(b[7, 5:min(n, 60)])
print("cycle per iteration (sm0 S-ready to S-ready): median", np.median(per_it))
print("softmax0 duration (sok->done): median", np.median(b[8, it] - b[7, it]))
print("softmax1 duration: median", np.median(b[11, it] - b[10, it]))
print("sm0 waiting for S (swait->sok): median", np.median(b[7, it] - b[6, it]))
print("mma waiting P0 (pwait->pok): median", np.median(b[1, it] - b[0, it]))
print("mma waiting P1: median", np.median(b[4, it] - b[3, it]))
print("P0 arrive -> mma sees it (sm0_done -> mma_pok0): median", np.median(b[1, it] - b[8, it]))
print("mma issue PV0+S0 -> sm0 S ready next (issued0[it] -> sok[it+1]): median", np.median(b[7, it + 1] - b[2, it]))
print("mma v wait: median", np.median(b[13, it] - b[12, it]))
