import sys, os, json, statistics
sys.path.insert(0, os.getcwd())
import torch, bench
from paper_2508_08192_b200 import _lib
from paper_2508_08192_b200.drafttree import tree_build
from paper_2508_08192_b200.attention import TreeVerifyAttention
from paper_2508_08192_b200.sharding import shard_for
_lib.load(); dev = torch.device("cuda", 0)
for ctx in (128, 1024, 8192):
    cfg = dict(bench.CONFIGS["c2"], ctx=ctx, V=1024)
    shard = shard_for(0, 1, cfg["Hq"], cfg["Hkv"], cfg["V"])
    x, R = bench.make_inputs(cfg, shard, dev)
    mask, _, _, _ = tree_build(x.parent, x.n_rows, x.ctx_len)
    for ctas in (0, 8, 16, 32, 148):
        attn = TreeVerifyAttention()
        call = lambda: attn(x.q, x.k_pool, x.v_pool, x.block_table, x.ctx_len, x.tree_k, x.tree_v, mask, x.n_rows, cfg["d"] ** -0.5, max_ctx=ctx, num_splits=ctas, kernel=1)
        call(); torch.cuda.synchronize()
        s = torch.cuda.Stream(); 
        with torch.cuda.stream(s): call()
        torch.cuda.synchronize()
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g): call()
        ts = []
        for _ in range(5):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            for _ in range(20): g.replay()
            e1.record(); torch.cuda.synchronize(); ts.append(e0.elapsed_time(e1) / 20 * 1e3)
        print(json.dumps({"ctx": ctx, "ctas": ctas, "us": statistics.median(ts)}))
