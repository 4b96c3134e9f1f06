"""Small launches of the pair attention kernel and the stochastic cluster
walk for compute-sanitizer (racecheck / synccheck / memcheck):
python tools/sanitize_cases.py attn|attn1|stoch"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import bench  # noqa: E402
from paper_2508_08192_b200 import _lib  # noqa: E402
from paper_2508_08192_b200.sharding import shard_for  # noqa: E402
from paper_2508_08192_b200.verify import TreeVerifier  # noqa: E402

_lib.load()
dev = torch.device("cuda", 0)
what = sys.argv[1] if len(sys.argv) > 1 else "attn"
if what == "attn":
    # 70B shapes, two sequences at 1k context: CTA-pair kernel, whole units + stream-K pieces + fix-up
    cfg = dict(bench.CONFIGS["c3"], B=2, ctx=1024, V=2048)
    x, R = bench.make_inputs(cfg, shard_for(0, 1, cfg["Hq"], cfg["Hkv"], cfg["V"]), dev)
    for splits in (0, 12):
        ver = TreeVerifier(scale=cfg["d"] ** -0.5, max_ctx=cfg["ctx"], num_splits=splits, kernel=1)
        out, lse, acc, terr = ver.step(x)
        torch.cuda.synchronize()
    print("attn ok", float(out.float().abs().mean()))
elif what == "attn1":
    # 1-CTA kernel (<= 128 query rows per KV head): the chain-3 tree, whole units + stream-K pieces + fix-up
    bench.TREE = bench.TREES["chain3"]
    cfg = dict(bench.CONFIGS["c3"], B=4, ctx=1024, V=2048)
    x, R = bench.make_inputs(cfg, shard_for(0, 1, cfg["Hq"], cfg["Hkv"], cfg["V"]), dev)
    for splits in (0, 40):
        ver = TreeVerifier(scale=cfg["d"] ** -0.5, max_ctx=cfg["ctx"], num_splits=splits, kernel=1)
        out, lse, acc, terr = ver.step(x)
        torch.cuda.synchronize()
    print("attn1 ok", float(out.float().abs().mean()))
else:
    # stochastic acceptance, lazy walk (8-CTA clusters) + validation scan, and eager
    cfg = dict(bench.CONFIGS["c5"], B=4, V=32768)
    x, R = bench.make_inputs(cfg, shard_for(0, 1, cfg["Hq"], cfg["Hkv"], cfg["V"]), dev, mode="stochastic")
    from paper_2508_08192_b200.sampling import StochasticAcceptor

    for lazy in (True, False):
        acc = StochasticAcceptor(lazy=lazy, levels=bench._tree_levels(tuple(bench._augment(bench.TREE))))
        res = acc(x.logits, x.draft_logits, 1.0, 0.9, x.parent, x.n_rows, x.tokens, seeds=x.seeds, steps=x.steps)
        torch.cuda.synchronize()
        res.raise_if_error()
    print("stoch ok", res.path_len.tolist())
