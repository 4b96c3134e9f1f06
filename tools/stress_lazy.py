"""Stress the lazy stochastic walk (cluster CTAs reading / writing the lazy
state): C5 inputs, many eager calls with the validation scan beside the walk
and per-call result comparison against the first call (determinism; a race
would show up as a mismatch or a launch failure).
usage: python tools/stress_lazy.py [iters]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import bench  # noqa: E402
from paper_2508_08192_b200 import _lib  # noqa: E402
from paper_2508_08192_b200.sampling import StochasticAcceptor, tree_levels  # noqa: E402
from paper_2508_08192_b200.sharding import shard_for  # noqa: E402

iters = int(sys.argv[1]) if len(sys.argv) > 1 else 200
_lib.load()
dev = torch.device("cuda", 0)
cfg = dict(bench.CONFIGS["c5"], ctx=64)
x, R = bench.make_inputs(cfg, shard_for(0, 1, cfg["Hq"], cfg["Hkv"], cfg["V"]), dev, mode="stochastic")
acc = StochasticAcceptor(lazy=True, levels=tree_levels(x.parent))


def run():
    r = acc(x.logits, x.draft_logits, bench.TEMPERATURE, bench.TOP_P, x.parent, x.n_rows, x.tokens, None,
            seeds=x.seeds, steps=x.steps)
    return (r.path.clone(), r.path_len.clone(), r.next_token.clone(), r.uniforms_used.clone(), r.err.clone())


ref = run()
torch.cuda.synchronize()
bad = 0
for i in range(iters):
    got = run()
    if i % 50 == 49:
        torch.cuda.synchronize()
    if not all(torch.equal(a, b) for a, b in zip(ref, got)):
        bad += 1
torch.cuda.synchronize()
print(f"stress: {iters} lazy calls, {bad} mismatches, err {int(ref[4][0])}, mean path {ref[1].float().mean().item():.3f}")
sys.exit(1 if bad else 0)
