"""Micro-benchmark of the tree-verify attention kernels alone (CUDA events,
median of repeated launch loops).  usage: python tools/attn_bench.py [config]
[--kernel K] [--ctas N]; env SDB_ATTN_EMU selects the exp2 emulation level."""
import argparse
import json
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

import bench  # noqa: E402
from paper_2508_08192_b200 import _lib  # noqa: E402
from paper_2508_08192_b200.drafttree import tree_build  # noqa: E402
from paper_2508_08192_b200.attention import TreeVerifyAttention  # noqa: E402
from paper_2508_08192_b200.sharding import shard_for  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("config", nargs="?", default="c3")
ap.add_argument("--kernel", type=int, default=1)
ap.add_argument("--ctas", type=int, default=0)
ap.add_argument("--gpus", type=int, default=1, help="simulate the per-GPU shard of a G-way KV-head split")
ap.add_argument("--iters", type=int, default=20)
ap.add_argument("--reps", type=int, default=5)
args = ap.parse_args()
cfg = bench.CONFIGS[args.config]
_lib.load()
dev = torch.device("cuda", 0)
shard = shard_for(0, args.gpus, cfg["Hq"], cfg["Hkv"], cfg["V"])
cfg2 = dict(cfg, V=1024)
x, R = bench.make_inputs(cfg2, shard, dev)
mask, _, _, _ = tree_build(x.parent, x.n_rows, x.ctx_len)
attn = TreeVerifyAttention()
call = lambda: attn(x.q, x.k_pool, x.v_pool, x.block_table, x.ctx_len, x.tree_k, x.tree_v, mask, x.n_rows,
                    cfg["d"] ** -0.5, max_ctx=cfg["ctx"], num_splits=args.ctas, kernel=args.kernel)
for _ in range(3):
    call()
torch.cuda.synchronize()
times = []
clk = bench.ClockSampler(0)
clk.__enter__()
for _ in range(args.reps):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(args.iters):
        call()
    e1.record()
    torch.cuda.synchronize()
    times.append(e0.elapsed_time(e1) / args.iters)
clk.__exit__()
ms = statistics.median(times)
from oracle import specdec_oracle as O  # noqa: E402  (mask popcount only)

anc = int(O.suffix_mask(tuple(bench._augment(bench.TREE64))).sum())
_, _, flops = bench.step_bytes_flops(cfg, shard, R, anc)
print(json.dumps({"config": args.config, "gpus": args.gpus, "kernel": args.kernel, "ctas": args.ctas,
                  "emu": os.environ.get("SDB_ATTN_EMU", "default"), "ms": ms, "tflops": flops / ms / 1e9,
                  "spread": [min(times), max(times)], "clocks": clk.summary()}))
