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

cfg = dict(bench.CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "c3"])
if os.environ.get("TRACE_TREE"):
    bench.TREE = bench.TREES[os.environ["TRACE_TREE"]]
if os.environ.get("TRACE_B"):
    cfg["B"] = int(os.environ["TRACE_B"])
lib = _lib.load()
dev = torch.device("cuda", 0)
shard = shard_for(0, 1, cfg["Hq"], cfg["Hkv"], cfg["V"])
x, R = bench.make_inputs(dict(cfg, V=1024), shard, dev)
mask, _, _, _ = tree_build(x.parent, x.n_rows, x.ctx_len)
attn = TreeVerifyAttention()
for _ in range(3):
    attn(x.q, x.k_pool, x.v_pool, x.block_table, x.ctx_len, x.tree_k, x.tree_v, mask, x.n_rows, cfg["d"] ** -0.5,
         max_ctx=cfg["ctx"], kernel=1, num_splits=int(os.environ.get("TRACE_CTAS", "0")))
torch.cuda.synchronize()
buf = np.zeros((24, 256), dtype=np.uint64)
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
if buf[19, 5]:
    k = np.arange(8, 50)
    print("tensor pipe: PV(n) done -> S(n+3) done: median", np.median(b[19, k + 3] - b[20, k]))
    print("tensor pipe: S(n+3) done -> PV(n+1) done: median", np.median(b[20, k + 1] - b[19, k + 3]))
    print("tensor pipe: PV(n) issue start (P seen) -> PV(n) done: median", np.median(b[20, k] - b[1, k]))
    print("tensor pipe: S(n+3) issued -> S(n+3) done: median", np.median(b[19, k + 3] - b[2, k]))
    print("tensor pipe: S(n) done -> softmax sees it: median", np.median(b[4, k] - b[19, k]))
    k5 = np.arange(8, 50)
    print("V(n+5) TMA issue - PV(n) done (slot reuse gate): median", np.median(b[16, k5 + 5] - b[20, k5]))
    print("V(n) TMA issue -> PV(n) issue start: median", np.median(b[1, k5] - b[16, k5]))
if buf[21, 1] and buf[23, 1]:
    for u in range(0, 4):
        if not buf[21, u]:
            break
        print(f"unit {u} end: bar.red+sums {int(buf[22, u]) - int(buf[21, u])}, o_last wait {int(buf[23, u]) - int(buf[22, u])}, "
              f"epilogue {int(buf[20, 129 + u]) - int(buf[23, u]) if buf[20, 129 + u] else None} (abs start {int(buf[21, u]) - int(t0)})")
if os.environ.get("TRACE_ROWS"):
    print("item: Vwait(18->0) Pwait(0->1) issue(1->2) loop(2->18') | sm: swait sok->done | S(n+3) lat")
    rows = [int(v) for v in os.environ.get("TRACE_ROWS").split(",")] if "," in os.environ.get("TRACE_ROWS") else list(range(8, 40))
    for k in rows:
        print(k, b[0, k] - b[18, k], b[1, k] - b[0, k], b[2, k] - b[1, k], b[18, k + 1] - b[2, k], "|",
              b[4, k] - b[3, k], b[5, k] - b[4, k], "|", b[4, k + 3] - b[2, k], "| abs: sok", b[4, k], "pok", b[1, k],
              "done", b[5, k])
it3 = np.arange(8, min(n, 200) - 3)
print("S(n+3) issued (after PV(n)) -> softmax sees S(n+3): median", np.median(b[4, it3 + 3] - b[2, it3]))
print("P(n) arrived -> softmax sees S(n+3): median", np.median(b[4, it3 + 3] - b[5, it3]))
if buf[16, 8]:
    print("V TMA issued -> MMA sees v_full: median", np.median(b[0, it] - b[16, it]))
    print("V TMA issued ahead of the MMA's V wait: median", np.median(b[18, it] - b[16, it]))
    print("MMA V wait (v_full): median", np.median(b[0, it] - b[18, it]))
    print("K TMA issue period: median", np.median(np.diff(b[17, 8:min(n, 200)])))
    print("V TMA issue period: median", np.median(np.diff(b[16, 8:min(n, 200)])))
print("period mma: median", np.median(np.diff(b[1, 8:min(n, 200)])))
print("softmax: S ready -> first chunk loaded: median", np.median(b[6, it] - b[4, it]))
print("softmax: chunk 0 loaded -> chunks 0, 1 exp'd: median", np.median(b[7, it] - b[6, it]))
print("softmax: chunks 2, 3 exp'd: median", np.median(b[15, it] - b[7, it]))
print("softmax: last store -> P arrived (wait::st, fence, arrive): median", np.median(b[5, it] - b[15, it]))
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
