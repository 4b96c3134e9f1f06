"""Times the stochastic validation scan alone (sdb_stochastic_validate) at C5:
python tools/scan_bench.py   (SDB_SCAN_TMA=0/1 selects the kernel)"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import bench  # noqa: E402
from paper_2508_08192_b200 import _lib  # noqa: E402
from paper_2508_08192_b200.sharding import shard_for  # noqa: E402

cfg = bench.CONFIGS["c5"]
lib = _lib.load()
dev = torch.device("cuda", 0)
x, R = bench.make_inputs(cfg, shard_for(0, 1, cfg["Hq"], cfg["Hkv"], cfg["V"]), dev, mode="stochastic")
err = torch.zeros(1, dtype=torch.int32, device=dev)
b, r, v = x.logits.shape


def call():
    _lib.check(lib.sdb_stochastic_validate(_lib.ptr(x.logits), _lib.ptr(x.draft_logits), b, r, v, _lib.ptr(x.parent),
                                           _lib.ptr(x.n_rows), None, 0, _lib.ptr(err), _lib.stream_ptr()), "validate")


for _ in range(3):
    call()
torch.cuda.synchronize()
ts = []
for _ in range(10):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    call()
    e1.record()
    torch.cuda.synchronize()
    ts.append(e0.elapsed_time(e1) * 1e3)
ts.sort()
print(json.dumps({"tma": os.environ.get("SDB_SCAN_TMA", "1"), "us": ts[len(ts) // 2], "min": ts[0], "err": int(err.item())}))
