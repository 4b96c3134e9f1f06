import os, sys
sys.path.insert(0, os.getcwd())
import torch, bench
from paper_2508_08192_b200 import _lib
from paper_2508_08192_b200.verify import TreeVerifier, _num_sms
from paper_2508_08192_b200.sharding import shard_for
_lib.load()
cfg = bench.CONFIGS["c3"]
sh = shard_for(0, 1, cfg["Hq"], cfg["Hkv"], cfg["V"])
x, R = bench.make_inputs(cfg, sh, torch.device("cuda", 0))
ver = TreeVerifier(scale=128 ** -0.5, max_ctx=8192)
b, r = x.parent.shape
print("auto reserve", ver._auto_reserve(x, b, r, _num_sms(torch.device("cuda", 0))), "scan_hides", ver._scan_hides(x, b, r, torch.device("cuda", 0)))
