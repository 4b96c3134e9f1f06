"""Lazy vs eager stochastic acceptance across batch sizes (C5 shapes: tree64,
V 128256, T 1, top-p 0.9; bench.make_inputs synthetic logits).  Device time
of CUDA-graph replays; one JSON line per batch.
usage: python tools/lazy_sweep.py [--batches 8,16,32,64]"""
import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

import bench  # noqa: E402
from paper_2508_08192_b200 import _lib  # noqa: E402
from paper_2508_08192_b200.sampling import StochasticAcceptor, tree_levels  # noqa: E402
from paper_2508_08192_b200.sharding import shard_for  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--batches", default="8,16,24,32,48,64")
ap.add_argument("--iters", type=int, default=10)
args = ap.parse_args()
_lib.load()
dev = torch.device("cuda", 0)
for B in [int(x) for x in args.batches.split(",")]:
    cfg = dict(bench.CONFIGS["c5"], B=B, ctx=64)
    shard = shard_for(0, 1, cfg["Hq"], cfg["Hkv"], cfg["V"])
    x, R = bench.make_inputs(cfg, shard, dev, mode="stochastic")
    levels = tree_levels(x.parent)
    out = {"batch": B}
    for lazy in (False, True):
        acc = StochasticAcceptor(lazy=lazy, levels=levels)
        fn = lambda: acc(x.logits, x.draft_logits, bench.TEMPERATURE, bench.TOP_P, x.parent, x.n_rows, x.tokens,
                         None, seeds=x.seeds, steps=x.steps)
        out["lazy_us" if lazy else "eager_us"] = bench.graph_time(fn, args.iters, torch.cuda.current_stream()) * 1e3
    print(json.dumps(out), flush=True)
    del x
    torch.cuda.empty_cache()
