"""Draft-side tree attention benchmark: one draft
round of the 63-node EAGLE tree at the Llama-3.3-70B attention shapes (B 32,
64q/8kv, d 128, ctx 8192 paged) = one rectangular call per depth (new nodes
attend the draft-cache prefix + carried/new suffix, engine.py:424-432).

Each depth re-reads the whole prefix KV (it is a different query set), so a
depth step is HBM-bound: algorithmic bytes = B*C*Hkv*d*2*2 (prefix K+V) +
B*n_new*Hq*d*2*2 (q, out) + B*total*Hkv*d*2*2 (suffix K+V).  Device time by
CUDA events around CUDA-graph replays; prints one JSON line.
usage: python tools/draft_bench.py [--kernel K] [--iters N]"""
import argparse
import json
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

import bench  # noqa: E402
from paper_2508_08192_b200 import _lib  # noqa: E402
from paper_2508_08192_b200.attention import TreeVerifyAttention  # noqa: E402
from paper_2508_08192_b200.drafttree import tree_build  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--kernel", type=int, default=1)
ap.add_argument("--iters", type=int, default=20)
ap.add_argument("--reps", type=int, default=5)
args = ap.parse_args()
_lib.load()
dev = torch.device("cuda", 0)
B, Hq, Hkv, d, C, bs = 32, 64, 8, 128, 8192, 64
tree = bench.TREE64  # realized draft nodes (no root row: the root is in the draft cache)
n = len(tree)
depth = []
for p in tree:
    depth.append(1 if p < 0 else depth[p] + 1)
pages = -(-C // bs)
nb = B * pages + 8
g = torch.Generator(device=dev).manual_seed(0)
kp = torch.randn((nb, Hkv, bs, d), generator=g, device=dev).to(torch.bfloat16)
vp = torch.randn((nb, Hkv, bs, d), generator=g, device=dev).to(torch.bfloat16)
table = torch.randperm(nb, generator=torch.Generator().manual_seed(1))[:B * pages].reshape(B, pages).to(
    torch.int32).to(dev)
q = torch.randn((B, n, Hq, d), generator=g, device=dev).to(torch.bfloat16)
sk = torch.randn((B, n, Hkv, d), generator=g, device=dev).to(torch.bfloat16)
sv = torch.randn((B, n, Hkv, d), generator=g, device=dev).to(torch.bfloat16)
ctx = torch.full((B,), C, dtype=torch.int32, device=dev)
par = torch.tensor([tree] * B, dtype=torch.int32, device=dev)
out = torch.empty_like(q)
lse = torch.empty((B, Hq, n), dtype=torch.float32, device=dev)
steps = []
for dep in range(1, max(depth) + 1):
    total = sum(1 for x in depth if x <= dep)
    q0 = sum(1 for x in depth if x < dep)
    nr = torch.full((B,), total, dtype=torch.int32, device=dev)
    mask, _, _, _ = tree_build(par, nr, ctx)
    steps.append(dict(depth=dep, q0=q0, total=total, nr=nr, mask=mask,
                      q0_t=torch.full((B,), q0, dtype=torch.int32, device=dev), attn=TreeVerifyAttention()))


def run_step(s):
    s["attn"](q, kp, vp, table, ctx, sk, sv, s["mask"], s["nr"], d ** -0.5, out=out, lse=lse, max_ctx=C,
              kernel=args.kernel, q_row0=s["q0_t"], max_q_nodes=s["total"] - s["q0"])


def graph_of(fn):
    st = torch.cuda.Stream()
    st.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(st):
        fn()
    torch.cuda.current_stream().wait_stream(st)
    torch.cuda.synchronize()
    gr = torch.cuda.CUDAGraph()
    with torch.cuda.graph(gr):
        fn()
    return gr


def time_graph(gr):
    times = []
    for _ in range(args.reps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(args.iters):
            gr.replay()
        e1.record()
        torch.cuda.synchronize()
        times.append(e0.elapsed_time(e1) / args.iters)
    return statistics.median(times)


peak = bench._measured_peaks()[0]
per = []
tot_bytes = 0
for s in steps:
    ms = time_graph(graph_of(lambda s=s: run_step(s)))
    n_new = s["total"] - s["q0"]
    byts = B * C * Hkv * d * 2 * 2 + B * n_new * Hq * d * 2 * 2 + B * s["total"] * Hkv * d * 2 * 2
    tot_bytes += byts
    per.append({"depth": s["depth"], "new_nodes": n_new, "keys_suffix": s["total"], "us": ms * 1e3,
                "gbs": byts / ms / 1e6, "frac_hbm": byts / ms / 1e6 / peak})
round_ms = time_graph(graph_of(lambda: [run_step(s) for s in steps]))
print(json.dumps({"bench": "draft-round tree attention (70B shapes, B32, ctx 8192, 63-node tree, 5 depths)",
                  "kernel": args.kernel, "round_us": round_ms * 1e3, "round_gbs": tot_bytes / round_ms / 1e6,
                  "round_frac_hbm": tot_bytes / round_ms / 1e6 / peak, "hbm_peak_gbs": peak, "depths": per}))
