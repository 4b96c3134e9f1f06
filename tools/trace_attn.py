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
names = ["mma_pwait", "mma_pok", "mma_issued", "sm_swait", "sm_sok", "sm_done"]
n = int((buf[4] > 0).sum())
print("items traced", n)
for it in range(min(n, 24)):
    print(it, " ".join(f"{names[e]}={b[e, it]:>8d}" for e in range(6)))
it = np.arange(8, min(n, 200))
print("item period (sm S-ready to S-ready): median", np.median(np.diff(b[4, 8:min(n, 200)])))
print("softmax duration (sok->done): median", np.median(b[5, it] - b[4, it]))
print("softmax WG item duration (sok->done): median", np.median(b[5, it] - b[4, it]))
print("softmax waiting for S (swait->sok): median", np.median(b[4, it] - b[3, it]))
print("mma waiting P (pwait->pok): median", np.median(b[1, it] - b[0, it]))
print("mma PV+S issue (pok->issued): median", np.median(b[2, it] - b[1, it]))
print("P arrive -> mma sees it: median", np.median(b[1, it] - b[5, it]))
print("mma issued(n) -> pwait(n+1) (V wait + loop): median", np.median(b[0, it + 1] - b[2, it]))
per = b[:, it]
print("period mma: median", np.median(np.diff(b[1, 8:min(n, 200)])))
print("softmax: S ready -> max pass done: median", np.median(b[6, it] - b[4, it]))
print("softmax: max done -> chain ok: median", np.median(b[7, it] - b[6, it]))
print("softmax: chain ok -> P arrived: median", np.median(b[5, it] - b[7, it]))
# kernel-level phases of worker 0 (clock64 of its SM)
e8 = int(buf[8, 0])
if e8:
    rel = lambda v: int(v) - e8
    print("entry -> setup done (barriers, TMEM alloc, cluster sync):", rel(buf[9, 0]))
    print("entry -> first S ready:", rel(buf[4, 0]) if buf[4, 0] else None)
    ends = [(i, rel(buf[10, i])) for i in range(256) if buf[10, i]]
    print("unit epilogues done (item index, cycles from entry):", ends[:8])
    print("entry -> softmax loop exit (thread 0):", rel(buf[11, 0]), " -> final cluster sync:", rel(buf[12, 0]))
# every worker (globaltimer ns): start / end spread
st = buf[13][buf[13] > 0].astype(np.int64)
en = buf[14][buf[14] > 0].astype(np.int64)
if len(st):
    t0 = st.min()
    print("workers", len(st), "start spread ns", int(st.max() - t0), "end: min", int(en.min() - t0), "median",
          int(np.median(en) - t0), "max", int(en.max() - t0))
