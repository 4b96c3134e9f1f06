"""Latency probe of the attention at bs 1 (8B shapes): device time of one
launch (CUDA graph replays) vs context length and persistent worker count."""
import json
import os
import statistics
import sys

sys.path.insert(0, os.getcwd())
import torch  # noqa: E402

import bench  # noqa: E402
from paper_2508_08192_b200 import _lib  # noqa: E402
from paper_2508_08192_b200.attention import TreeVerifyAttention  # noqa: E402
from paper_2508_08192_b200.drafttree import tree_build  # noqa: E402
from paper_2508_08192_b200.sharding import shard_for  # noqa: E402

_lib.load()
dev = torch.device("cuda", 0)
ctxs = [int(c) for c in (sys.argv[1].split(",") if len(sys.argv) > 1 else ["128", "1024", "8192"])]
ctas_list = [int(c) for c in (sys.argv[2].split(",") if len(sys.argv) > 2 else ["0", "1", "2", "8", "16", "32"])]
for ctx in ctxs:
    cfg = dict(bench.CONFIGS["c2"], ctx=ctx, V=1024)
    shard = shard_for(0, 1, cfg["Hq"], cfg["Hkv"], cfg["V"])
    x, R = bench.make_inputs(cfg, shard, dev)
    mask, _, _, _ = tree_build(x.parent, x.n_rows, x.ctx_len)
    for ctas in ctas_list:
        attn = TreeVerifyAttention()

        def call():
            attn(x.q, x.k_pool, x.v_pool, x.block_table, x.ctx_len, x.tree_k, x.tree_v, mask, x.n_rows,
                 cfg["d"] ** -0.5, max_ctx=ctx, num_splits=ctas, kernel=1)

        call()
        torch.cuda.synchronize()
        s = torch.cuda.Stream()
        with torch.cuda.stream(s):
            call()
        torch.cuda.synchronize()
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g):
            call()
        ts = []
        for _ in range(5):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            for _ in range(20):
                g.replay()
            e1.record()
            torch.cuda.synchronize()
            ts.append(e0.elapsed_time(e1) / 20 * 1e3)
        print(json.dumps({"ctx": ctx, "ctas": ctas, "us": round(statistics.median(ts), 2)}))
