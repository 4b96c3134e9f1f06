"""R = 65 (64 drafts + root) split experiment: the pair kernel on nodes
[0, 64) (512 rows per KV head = two whole 256-row tiles) with P CTA pairs,
and node 64 (8 rows per KV head) by the SIMT kernel on a forked stream in
the SMs the pair kernel leaves.  Device time of CUDA-graph replays; checks
the split result against the one-call result."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import bench  # noqa: E402
from paper_2508_08192_b200 import _lib  # noqa: E402
from paper_2508_08192_b200.attention import TreeVerifyAttention  # noqa: E402
from paper_2508_08192_b200.drafttree import tree_build  # noqa: E402
from paper_2508_08192_b200.sharding import shard_for  # noqa: E402

_lib.load()
dev = torch.device("cuda", 0)
bench.TREE = bench.TREE64 + [0]
cfg = dict(bench.CONFIGS["c3"], V=1024)
shard = shard_for(0, 1, cfg["Hq"], cfg["Hkv"], cfg["V"])
x, R = bench.make_inputs(cfg, shard, dev)
assert R == 65
B = cfg["B"]
mask, _, _, _ = tree_build(x.parent, x.n_rows, x.ctx_len)
scale = cfg["d"] ** -0.5
base = (x.q, x.k_pool, x.v_pool, x.block_table, x.ctx_len, x.tree_k, x.tree_v, mask, x.n_rows, scale)
out_ref = torch.empty_like(x.q)
lse_ref = torch.empty((B, cfg["Hq"], R), dtype=torch.float32, device=dev)
out = torch.empty_like(x.q)
lse = torch.empty_like(lse_ref)
q64 = torch.full((B,), 64, dtype=torch.int32, device=dev)
full = TreeVerifyAttention()
main = TreeVerifyAttention()
tail = TreeVerifyAttention()
side = torch.cuda.Stream()


def run_full():
    full(*base, out=out_ref, lse=lse_ref, max_ctx=cfg["ctx"])


def run_split(pairs, splits, tail_first=False):
    def f():
        cur = torch.cuda.current_stream()
        ev = torch.cuda.Event()
        ev.record(cur)
        side.wait_event(ev)

        def t():
            with torch.cuda.stream(side):
                tail(*base, out=out, lse=lse, max_ctx=cfg["ctx"], kernel=2, q_row0=q64, max_q_nodes=1,
                     num_splits=splits)
        if tail_first:
            t()
        main(*base, out=out, lse=lse, max_ctx=cfg["ctx"], max_q_nodes=64, num_splits=pairs)
        if not tail_first:
            t()
        ev2 = torch.cuda.Event()
        ev2.record(side)
        cur.wait_event(ev2)
    return f


def run_tail(splits):
    def f():
        tail(*base, out=out, lse=lse, max_ctx=cfg["ctx"], kernel=2, q_row0=q64, max_q_nodes=1, num_splits=splits)
    return f


def run_main(pairs):
    def f():
        main(*base, out=out, lse=lse, max_ctx=cfg["ctx"], max_q_nodes=64, num_splits=pairs)
    return f


res = {"full_us": bench.graph_time(run_full, 20, torch.cuda.current_stream()) * 1e3}
for s in (0, 4, 8, 16):
    res[f"tail_s{s}_us"] = bench.graph_time(run_tail(s), 20, torch.cuda.current_stream()) * 1e3
for p in (62, 66, 70, 74):
    res[f"main_p{p}_us"] = bench.graph_time(run_main(p), 20, torch.cuda.current_stream()) * 1e3
for p in (62, 66, 70):
    for s in (0, 4, 8):
        for tf in (False, True):
            res[f"split_p{p}_s{s}{'_tf' if tf else ''}_us"] = bench.graph_time(
                run_split(p, s, tf), 20, torch.cuda.current_stream()) * 1e3
torch.cuda.synchronize()
run_full()
run_split(66, 0)()
torch.cuda.synchronize()
d = (out.float() - out_ref.float()).abs()
res["max_abs_diff_main_rows"] = float(d[:, :64].max())
res["max_abs_diff_tail_rows"] = float(d[:, 64:].max())
res["max_lse_diff"] = float((lse - lse_ref).abs().max())
print(json.dumps(res, indent=0))
