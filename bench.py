"""Tree-verify benchmark (BASELINE.json metric: tree-verify us/step & HBM GB/s).

Workload (N = 1): Llama-3.3-70B attention shapes (configs[2]) -- B = 32,
64 q / 8 kv heads, d = 128, the 64-row EAGLE tree of SURVEY.md 8(d) (63 drafts
+ root), ctx 8192 in bf16 pages of 64, greedy acceptance over fp32 logits of
V = 128,256.  One step = tree_build + paged GQA tree attention (prefix +
masked suffix + LSE merge) + acceptance + KV compaction for one layer.
N > 1: KV heads (and their q heads) and the vocabulary are sharded over the
ranks (strong scaling); one NCCL all-reduce(MAX) of packed argmax keys per
step.  Synthetic seeded inputs; working set (KV + logits, ~2.1 GB per GPU at
N = 1) far exceeds the 126 MB L2, so every step streams from HBM.

`--impl reference` times the reference algorithm on the host (the numpy
oracle port: the reference is pure Python/numpy, nothing compiles) on a
bounded sample and extrapolates exactly (the reference loops sequences and
heads independently, engine.py:581-582).
"""

from __future__ import annotations

import argparse
import json
import os
import statistics
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "tree-verify μs/step & HBM GB/s (% of 8 TB/s) at bs1–64, 8k ctx, 1/2/4/8 GPU"

# the 63-node EAGLE tree of SURVEY.md 8(d) (R = 64 rows with the root); the
# mandatory R = 65 variant appends a 7th child of node 0 (`--tree 65`)
TREE64 = [-1, -1, -1, -1, -1, -1, -1, -1, 0, 0, 0, 0, 0, 0, 1, 1, 1, 1, 1, 2, 2, 2, 2, 3, 3, 3, 4, 4, 5, 5, 6, 7,
          8, 8, 8, 8, 9, 9, 9, 10, 10, 10, 11, 11, 12, 13, 14, 15, 32, 32, 32, 33, 33, 34, 34, 35, 36, 37, 48, 48, 49,
          50, 51]

CONFIGS = {
    # name: (B, Hq, Hkv, d, ctx, block_size, vocab, tree)
    "c3": dict(workload="llama-3.3-70b-attn bs32 ctx8192 tree64 greedy", B=32, Hq=64, Hkv=8, d=128, ctx=8192, bs=64,
               V=128256),
    "c2": dict(workload="llama-3.1-8b-attn bs1 ctx8192 tree64 greedy", B=1, Hq=32, Hkv=8, d=128, ctx=8192, bs=64,
               V=128256),
    "c4": dict(workload="llama-3.1-405b-attn bs64 ctx32768 tree64 greedy", B=64, Hq=128, Hkv=8, d=128, ctx=32768,
               bs=64, V=128256),
    # acceptance only (configs[4]): stochastic top-p MSS over 128k logits
    "c5": dict(workload="stochastic top-p acceptance bs64 tree64 V128256 T1 p0.9", B=64, Hq=64, Hkv=8, d=128,
               ctx=0, bs=64, V=128256, accept_only=True, mode="stochastic"),
}
TEMPERATURE, TOP_P = 1.0, 0.9
# HBM-bound contrast trees of SURVEY.md 8(d) at the C3 shapes: chain-3
# (build_chain(3), drafttree.py:60-63; R = 4, R*g = 32) and the reference's
# N8 tree (R = 9, R*g = 72)
TREES = {"64": TREE64, "65": TREE64 + [0], "chain3": [-1, 0, 1], "n8": [-1, -1, 0, 0, 1, 2, 2, 5]}
TREE = TREE64  # set from --tree


def _augment(parent):
    return [-1] + [0 if p == -1 else p + 1 for p in parent]


def _ancestor_pairs(aug):
    """Number of (row, key) pairs of the ancestor-or-self tree mask."""
    depth = []
    for p in aug:
        depth.append(1 if p < 0 else depth[p] + 1)
    return sum(depth)


def _tree_levels(aug):
    depth = []
    for p in aug:
        depth.append(0 if p < 0 else depth[p] + 1)
    return max(depth) + 1


def _measured_peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            pk = json.load(f)
        return pk["hbm_gbs"], pk["bf16_tflops"], "measured"
    except Exception:
        return 6650.0, 1590.0, "fallback"


class ClockSampler:
    """Polls NVML SM clock + throttle reasons in a thread during the timed region."""

    REASONS = {0x8: "hw_slowdown", 0x40: "hw_thermal_slowdown", 0x20: "sw_thermal_slowdown", 0x4: "sw_power_cap",
               0x80: "hw_power_brake_slowdown", 0x1: "gpu_idle"}

    def __init__(self, device_index):
        self.samples, self.reasons, self.max_mhz = [], set(), None
        self._stop = threading.Event()
        try:
            import pynvml

            pynvml.nvmlInit()
            self._nvml = pynvml
            self._h = pynvml.nvmlDeviceGetHandleByIndex(device_index)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self._h, pynvml.NVML_CLOCK_SM)
        except Exception:
            self._nvml = None

    def _run(self):
        while not self._stop.is_set():
            try:
                self.samples.append(self._nvml.nvmlDeviceGetClockInfo(self._h, self._nvml.NVML_CLOCK_SM))
                r = self._nvml.nvmlDeviceGetCurrentClocksEventReasons(self._h)
                for bit, name in self.REASONS.items():
                    if r & bit and name != "gpu_idle":
                        self.reasons.add(name)
            except Exception:
                pass
            time.sleep(0.002)

    def __enter__(self):
        if self._nvml is not None:
            self._t = threading.Thread(target=self._run, daemon=True)
            self._t.start()
        return self

    def __exit__(self, *a):
        self._stop.set()
        if self._nvml is not None:
            self._t.join()

    def summary(self):
        return {"sm_mhz": statistics.median(self.samples) if self.samples else None, "sm_max_mhz": self.max_mhz,
                "reasons": sorted(self.reasons), "samples": len(self.samples)}


def make_inputs(cfg, shard, device, seed=0, mode="greedy"):
    """Seeded synthetic inputs for one rank's shard (KV heads, vocab range)."""
    import torch

    from paper_2508_08192_b200.verify import StepInputs

    g = torch.Generator(device=device)
    g.manual_seed(seed)
    B, Hq, Hkv, d, C, bs, V = (cfg[k] for k in ("B", "Hq", "Hkv", "d", "ctx", "bs", "V"))
    aug = _augment(TREE)
    R = len(aug)
    hkv_l, hq_l = shard.n_kv, shard.n_q
    pages = -(-(C + R) // bs)
    nb = B * pages + 8
    # identical page permutation on every rank (same block table)
    perm = torch.randperm(nb, generator=torch.Generator().manual_seed(seed + 1)).to(torch.int32)
    if os.environ.get("SDB_BENCH_PAGES") == "seq":  # A/B: each sequence's pages contiguous in the pool
        perm = torch.arange(nb, dtype=torch.int32)
    table = perm[:B * pages].reshape(B, pages).to(device)

    def randn(*shape, dtype=torch.bfloat16, std=1.0, gen=g):
        return (torch.randn(*shape, generator=gen, device=device) * std).to(dtype)

    # full-head tensors are drawn per KV-head slice so shards see the same data
    def per_head(shape_fn, n_total, lo, hi, dtype, seed_off):
        parts = []
        for h in range(lo, hi):
            gh = torch.Generator(device=device)
            gh.manual_seed(seed * 1000 + seed_off * 97 + h)
            parts.append((torch.randn(*shape_fn(), generator=gh, device=device)).to(dtype))
        return parts

    kp = torch.stack(per_head(lambda: (nb, bs, d), Hkv, shard.kv_lo, shard.kv_hi, torch.bfloat16, 1), dim=1)
    vp = torch.stack(per_head(lambda: (nb, bs, d), Hkv, shard.kv_lo, shard.kv_hi, torch.bfloat16, 2), dim=1)
    q = torch.stack(per_head(lambda: (B, R, d), Hq, shard.q_lo, shard.q_hi, torch.bfloat16, 3), dim=2)
    tk = torch.stack(per_head(lambda: (B, R, d), Hkv, shard.kv_lo, shard.kv_hi, torch.bfloat16, 4), dim=2)
    tv = torch.stack(per_head(lambda: (B, R, d), Hkv, shard.kv_lo, shard.kv_hi, torch.bfloat16, 5), dim=2)
    # logits: the full vocab on every rank (setup only), then this rank's slice
    gl = torch.Generator(device=device)
    gl.manual_seed(seed + 7)
    logits_full = torch.randn(B, R, V, generator=gl, device=device) * 2.0
    am = logits_full.argmax(dim=-1)  # lowest index on ties
    par = torch.tensor([aug] * B, dtype=torch.int32, device=device)
    tokens = torch.zeros((B, R), dtype=torch.int32, device=device)
    rnd = torch.rand((B, R), generator=gl, device=device)
    rtok = torch.randint(0, V, (B, R), generator=gl, device=device)
    parent_row = par.clamp(min=0).long()
    want = torch.gather(am, 1, parent_row)
    tokens = torch.where(rnd < 0.6, want, rtok).to(torch.int32)
    draft = seeds = steps = None
    if mode == "stochastic":
        # draft = target + N(0, 0.5^2); node tokens sampled from
        # the parent's draft q (stochastic drafting, engine.py:393-394)
        draft_full = logits_full + 0.5 * torch.randn(B, R, V, generator=gl, device=device)
        qd = torch.softmax(draft_full / TEMPERATURE, dim=-1)
        samp = torch.multinomial(qd.reshape(B * R, V), 1, generator=gl).reshape(B, R)
        tokens = torch.gather(samp, 1, parent_row).to(torch.int32)
        del qd
        draft = draft_full[:, :, shard.v_lo:shard.v_hi].contiguous()
        del draft_full
        seeds = torch.arange(B, dtype=torch.int64, device=device) + 1000 * (seed + 1)  # sampler.seed + seq
        steps = torch.full((B,), 2 * 7 + 2, dtype=torch.int64, device=device)          # 2*round + 2
    tokens[:, 0] = 0
    logits = logits_full[:, :, shard.v_lo:shard.v_hi].contiguous()
    del logits_full
    x = StepInputs(parent=par, n_rows=torch.full((B,), R, dtype=torch.int32, device=device),
                   ctx_len=torch.full((B,), C, dtype=torch.int32, device=device), tokens=tokens, q=q.contiguous(),
                   tree_k=tk.contiguous(), tree_v=tv.contiguous(), logits=logits, k_pool=kp.contiguous(),
                   v_pool=vp.contiguous(), block_table=table, draft_logits=draft, seeds=seeds, steps=steps)
    return x, R


def step_bytes_flops(cfg, shard, R, anc_pairs):
    B, d, C, V = cfg["B"], cfg["d"], cfg["ctx"], shard.n_vocab
    hq, hkv = shard.n_q, shard.n_kv
    s = 2
    attn_bytes = (B * C * hkv * d * 2 * s + B * R * hq * d * s + B * R * hkv * d * 2 * s + B * R * hq * d * s
                  + 4 * B * hq * R + 4 * B * (-(-C // cfg["bs"])))
    accept_bytes = B * R * V * 4
    attn_flops = 4.0 * d * hq * B * (R * C + anc_pairs)
    return attn_bytes, accept_bytes, attn_flops


def cpu_sample(cfg, seed=0, mode="greedy"):
    """Reference algorithm (numpy oracle port) on a bounded sample of the
    workload: 1 sequence x 1 KV head group for attention, 1 sequence for
    acceptance (greedy: argmax target_dist per row + walk; stochastic:
    top-p target_dist per row, draft q per parent row, mss_verify).  Returns
    (attention seconds, acceptance seconds, attention and acceptance
    extrapolation factors)."""
    import numpy as np

    from oracle import specdec_oracle as O

    rng = np.random.default_rng(seed)
    B, Hq, Hkv, d, C, bs, V = (cfg[k] for k in ("B", "Hq", "Hkv", "d", "ctx", "bs", "V"))
    g = Hq // Hkv
    aug = tuple(_augment(TREE))
    R = len(aug)
    parent = tuple(p - 1 if p > 0 else -1 for p in aug[1:])
    ta = 0.0
    if not cfg.get("accept_only"):
        pages = -(-(C + R) // bs)

        def bf(x):
            return x.astype(np.float32).astype(np.float64)

        kp = bf(rng.normal(size=(pages + 1, 1, bs, d)))
        vp = bf(rng.normal(size=(pages + 1, 1, bs, d)))
        table = rng.permutation(pages + 1)[:pages]
        q = bf(rng.normal(size=(R, g * d)))
        tk = bf(rng.normal(size=(R, d)))
        tv = bf(rng.normal(size=(R, d)))
        t0 = time.perf_counter()
        ck = O.paged_gather(kp, table, C)
        cv = O.paged_gather(vp, table, C)
        O.tree_attention(q, ck, cv, tk, tv, aug, d ** -0.5, g, 1)
        ta = time.perf_counter() - t0
    logits = (2.0 * rng.normal(size=(R, V))).astype(np.float32)
    toks = rng.integers(0, V, size=R)
    t1 = time.perf_counter()
    if mode == "greedy":
        dists = [O.target_dist(logits[i], 0.0, 1.0) for i in range(R)]
        am = [int(np.argmax(dd)) for dd in dists]
        O.greedy_walk(parent, toks[1:], am)
    else:
        draft = (logits + 0.5 * rng.normal(size=(R, V))).astype(np.float32)
        tdists = [O.target_dist(logits[i].astype(np.float64), TEMPERATURE, TOP_P) for i in range(R)]
        qs = {p: O.target_dist(draft[p].astype(np.float64), TEMPERATURE, 1.0) for p in set(aug[1:])}
        O.mss_verify(parent, toks[1:], [qs[p] for p in aug[1:]], tdists, O.uniform_row(seed, 16, R))
    tacc = time.perf_counter() - t1
    return ta, tacc, B * Hkv, B


def parity_sample(cfg, x, out, lse, acc, mode, aug):
    """Check one sampled sequence of the measured run against the CPU oracle
    (the cpu_baseline leg's restatement): accepted path / bonus token /
    uniforms used, and out / LSE of one (sequence, KV head) slice in float64
    (bf16 tolerances of tests/test_gpu_benched_configs.py)."""
    import numpy as np

    from oracle import specdec_oracle as O

    b = cfg["B"] // 2
    R = len(aug)
    raw = tuple(p - 1 if p > 0 else -1 for p in aug[1:])
    tokens = x.tokens[b].cpu().numpy()
    if mode == "greedy":
        want = O.greedy_walk(raw, tokens[1:], np.argmax(x.logits[b].cpu().numpy(), axis=-1))
    else:
        qmemo = {}

        def qdist(c):
            row = aug[1 + c]
            if row not in qmemo:
                qmemo[row] = O.target_dist(x.draft_logits[b, row].double().cpu().numpy(), TEMPERATURE, 1.0)
            return qmemo[row]

        uni = O.rank_sliced_uniforms(int(x.seeds[b]), int(x.steps[b]), 1, R)[0]
        w = O.mss_verify(raw, tokens[1:], qdist,
                         lambda i: O.target_dist(x.logits[b, i].double().cpu().numpy(), TEMPERATURE, TOP_P), uni)
        want = (w[0], w[1], w[3])
    plen = int(acc.path_len[b])
    got = ([int(a) for a in acc.path[b, :plen].cpu()], int(acc.next_token[b]), int(acc.uniforms_used[b]))
    res = {"sequence": b, "accept_exact": got == (list(want[0]), int(want[1]), int(want[2]))}
    if out is not None:
        g = cfg["Hq"] // cfg["Hkv"]
        f64 = lambda t: t.float().cpu().numpy().astype(np.float64)
        c = int(x.ctx_len[b])
        n_pages = -(-c // x.k_pool.shape[2])
        pages = x.block_table[b, :n_pages].long()
        wo, wl = O.tree_verify_attention_batch(f64(x.q[b:b + 1, :, :g]), f64(x.k_pool[pages][:, :1]),
                                               f64(x.v_pool[pages][:, :1]), np.arange(n_pages)[None],
                                               np.array([c]), f64(x.tree_k[b:b + 1, :, :1]),
                                               f64(x.tree_v[b:b + 1, :, :1]), [aug], cfg["d"] ** -0.5)
        err_o = np.abs(out[b, :, :g].float().cpu().numpy() - wo[0])
        err_l = float(np.abs(lse[b, :g].cpu().numpy() - wl[0]).max())
        res.update(kv_head=0, out_max_abs=float(err_o.max()), out_mean_abs=float(err_o.mean()), lse_max_abs=err_l,
                   attn_ok=bool(err_o.max() < 2e-2 and err_o.mean() < 2e-3 and err_l < 2e-3))
    res["ok"] = bool(res["accept_exact"] and res.get("attn_ok", True))
    return res


REF_DIR = os.path.join(ROOT, "baseline", "_ref")


def load_reference():
    """The unmodified reference package installed in baseline/_ref (pip
    --target, gitignored, shipped with the snapshot), or None."""
    if not os.path.isdir(os.path.join(REF_DIR, "specdec")):
        return None
    import tempfile

    os.environ.setdefault("NUMBA_CACHE_DIR", os.path.join(tempfile.gettempdir(), "sdb_numba_cache"))
    if REF_DIR not in sys.path:
        sys.path.insert(0, REF_DIR)
    import specdec
    import specdec.attention
    import specdec.engine
    import specdec.kernels
    import specdec.sampling

    return specdec


def reference_sample(ref, cfg, seed=0, mode="greedy"):
    """The STOCK reference path on a bounded sample of the workload: one
    sequence x one KV-head group of the attention through
    specdec.attention.tree_attention (kernels.attend_heads under the numba and
    the numpy backends; GQA by repeating the KV head), and one
    sequence of acceptance: specdec.sampling.target_dist for every row (+ the
    draft q of every parent row) and mss_verify (sampling.py:87-202).
    Returns {"attn_numba": s, "attn_numpy": s, "accept": s}."""
    import numpy as np

    rng = np.random.default_rng(seed)
    B, Hq, Hkv, d, C, V = (cfg[k] for k in ("B", "Hq", "Hkv", "d", "ctx", "V"))
    g = Hq // Hkv
    tree = ref.drafttree.TreeSpec(tuple(TREE))
    aug = ref.engine._augment(tree)
    R = aug.n_nodes
    out = {}
    if not cfg.get("accept_only"):
        def bf(x):
            return np.asarray(x, dtype=np.float32).astype(np.float64)

        q = bf(rng.normal(size=(R, g * d)))
        ck = np.repeat(bf(rng.normal(size=(C, 1, d))), g, axis=1).reshape(C, g * d)
        cv = np.repeat(bf(rng.normal(size=(C, 1, d))), g, axis=1).reshape(C, g * d)
        tk = np.repeat(bf(rng.normal(size=(R, 1, d))), g, axis=1).reshape(R, g * d)
        tv = np.repeat(bf(rng.normal(size=(R, 1, d))), g, axis=1).reshape(R, g * d)
        for backend in ("numba", "numpy"):
            prev = ref.kernels.set_backend(backend)
            try:
                t0 = time.perf_counter()
                ref.attention.tree_attention(q, ck, cv, tk, tv, aug, d ** -0.5, n_heads=g)
                out["attn_" + backend] = time.perf_counter() - t0
            finally:
                ref.kernels.set_backend(prev)
    logits = (2.0 * rng.normal(size=(R, V))).astype(np.float32).astype(np.float64)
    draft = logits + 0.5 * rng.normal(size=(R, V))
    T, top_p = (0.0, 1.0) if mode == "greedy" else (TEMPERATURE, TOP_P)
    t1 = time.perf_counter()
    tdists = [ref.sampling.target_dist(logits[i], T, top_p) for i in range(R)]
    qrow = {p_: ref.sampling.target_dist(draft[p_], T, 1.0) for p_ in set(aug.parent[1:])}
    node_dists = tuple(qrow[aug.parent[1 + c]] for c in range(tree.n_nodes))
    tokens = tuple(int(rng.integers(V)) for _ in range(tree.n_nodes))
    res = ref.sampling.mss_verify(ref.sampling.DraftResult(tree, tokens, node_dists), tdists,
                                  ref.sampling.rank_sliced_uniforms(seed, 16, 1, R + 1)[0],
                                  "greedy_children" if mode == "greedy" else "stochastic")
    out["accept"] = time.perf_counter() - t1
    out["accepted"] = len(res.accepted_path)
    return out


def blas_threads():
    try:
        from threadpoolctl import threadpool_info

        return max([i.get("num_threads", 1) for i in threadpool_info()] or [1])
    except Exception:
        return os.cpu_count() or 1


def _sample_desc(cfg, mode, cores):
    acc = ("greedy target_dist + argmax walk" if mode == "greedy"
           else f"top-p {TOP_P} target_dist per row + draft q per parent row + mss_verify")
    att = ("" if cfg.get("accept_only") else
           f"1 sequence x 1 KV-head group ({cfg['Hq'] // cfg['Hkv']} q heads) of the attention extrapolated "
           f"x{cfg['B'] * cfg['Hkv']}, + ")
    return f"{att}{acc} for 1 sequence x{cfg['B']}; numpy float64 oracle port, {cores} BLAS threads, extrapolated"


_REF = {}


def _ref_worker_init(cfg, mode, tree, seed, backend="numpy"):
    """Pool worker: one BLAS thread, the stock reference imported, one unit's
    inputs drawn once (the reference's cost does not depend on the values)."""
    import numpy as np

    try:
        from threadpoolctl import threadpool_limits

        threadpool_limits(1)
    except Exception:  # noqa: BLE001 - threadpoolctl is optional
        pass
    global TREE
    TREE = tree
    ref = load_reference()
    ref.kernels.set_backend(backend)
    rng = np.random.default_rng(seed)
    Hq, Hkv, d, C, V = (cfg[k] for k in ("Hq", "Hkv", "d", "ctx", "V"))
    g = Hq // Hkv
    spec = ref.drafttree.TreeSpec(tuple(tree))
    aug = ref.engine._augment(spec)
    R = aug.n_nodes
    st = {"ref": ref, "aug": aug, "spec": spec, "g": g, "d": d, "mode": mode, "seed": seed}
    if not cfg.get("accept_only"):
        def bf(x):
            return np.asarray(x, dtype=np.float32).astype(np.float64)

        st["q"] = bf(rng.normal(size=(R, g * d)))
        st["ck"] = np.repeat(bf(rng.normal(size=(C, 1, d))), g, axis=1).reshape(C, g * d)
        st["cv"] = np.repeat(bf(rng.normal(size=(C, 1, d))), g, axis=1).reshape(C, g * d)
        st["tk"] = np.repeat(bf(rng.normal(size=(R, 1, d))), g, axis=1).reshape(R, g * d)
        st["tv"] = np.repeat(bf(rng.normal(size=(R, 1, d))), g, axis=1).reshape(R, g * d)
    st["logits"] = (2.0 * rng.normal(size=(R, V))).astype(np.float32).astype(np.float64)
    st["draft"] = st["logits"] + 0.5 * rng.normal(size=(R, V))
    st["tokens"] = tuple(int(t) for t in rng.integers(V, size=spec.n_nodes))
    _REF.update(st)


def _ref_attn_unit(_i):
    """One (sequence, KV head) unit of the stock tree attention
    (specdec.attention.tree_attention, attention.py:131-151)."""
    s = _REF
    s["ref"].attention.tree_attention(s["q"], s["ck"], s["cv"], s["tk"], s["tv"], s["aug"], s["d"] ** -0.5,
                                      n_heads=s["g"])
    return 0


def _ref_accept_seq(_i):
    """One sequence of stock acceptance: target_dist of every row, the draft
    q of every parent row, mss_verify (sampling.py:87-202)."""
    s = _REF
    ref, aug, spec = s["ref"], s["aug"], s["spec"]
    T, top_p = (0.0, 1.0) if s["mode"] == "greedy" else (TEMPERATURE, TOP_P)
    tdists = [ref.sampling.target_dist(s["logits"][i], T, top_p) for i in range(aug.n_nodes)]
    qrow = {p_: ref.sampling.target_dist(s["draft"][p_], T, 1.0) for p_ in set(aug.parent[1:])}
    node_dists = tuple(qrow[aug.parent[1 + c]] for c in range(spec.n_nodes))
    res = ref.sampling.mss_verify(ref.sampling.DraftResult(spec, s["tokens"], node_dists), tdists,
                                  ref.sampling.rank_sliced_uniforms(s["seed"], 16, 1, aug.n_nodes + 1)[0],
                                  "greedy_children" if s["mode"] == "greedy" else "stochastic")
    return len(res.accepted_path)


def _host_cores():
    try:
        return len(os.sched_getaffinity(0))
    except Exception:  # noqa: BLE001
        return os.cpu_count() or 1


def reference_pool(cfg, mode, steps, warmup, start="fork"):
    """The stock reference path (baseline/_ref) on a pool of one-BLAS-thread
    processes over every host core: each step runs the step's (sequence, KV
    head) tree_attention units and its sequences' target_dist + mss_verify
    (the reference loops them independently, engine.py:581-582; attention per
    KV head), so the pool's wall time is the reference's best multi-core step.
    The whole step when it fits twice a 3 s budget, else a fixed share of the
    units scaled to the batch.  Returns (seconds per step, cores, sample
    description, extra fields) or None when baseline/_ref is absent."""
    ref = load_reference()
    if ref is None:
        return None
    import multiprocessing as mp

    cores = _host_cores()
    f_attn = 0 if cfg.get("accept_only") else cfg["B"] * cfg["Hkv"]
    f_acc = cfg["B"]
    # both stock attention backends timed on one unit (numba JIT warmed first); the faster runs
    one = reference_sample(ref, cfg, seed=10_000, mode=mode)
    one = reference_sample(ref, cfg, seed=10_001, mode=mode)
    backends = {k[len("attn_"):]: v for k, v in one.items() if k.startswith("attn_")}
    backend = min(backends, key=backends.get) if backends else "numpy"
    _REF["backend"] = backend
    t_unit = backends.get(backend, 0.0)
    budget = 3.0  # seconds of pool wall time per step
    # the whole step when it fits twice the budget, else a fixed share
    n_attn = (f_attn if t_unit * f_attn <= 2 * budget * cores
              else max(cores, int(budget * cores / max(t_unit, 1e-9))))
    n_acc = (f_acc if one["accept"] * f_acc <= 2 * budget * cores
             else max(cores, int(budget * cores / max(one["accept"], 1e-9))))
    n_attn, n_acc = min(n_attn, f_attn), min(n_acc, f_acc)
    ctx = mp.get_context(start)
    times = []
    with ctx.Pool(cores, initializer=_ref_worker_init, initargs=(cfg, mode, list(TREE), 0, backend)) as pool:
        for i in range(warmup + steps):
            t0 = time.perf_counter()
            if n_attn:
                pool.map(_ref_attn_unit, range(n_attn), chunksize=1)
            t1 = time.perf_counter()
            pool.map(_ref_accept_seq, range(n_acc), chunksize=1)
            t2 = time.perf_counter()
            if i >= warmup:
                times.append(((t1 - t0) * (f_attn / n_attn if n_attn else 0.0), (t2 - t1) * f_acc / n_acc))
    attn_s = statistics.mean(t[0] for t in times)
    acc_s = statistics.mean(t[1] for t in times)
    full = n_attn == f_attn and n_acc == f_acc
    sample = (f"stock specdec (baseline/_ref), {backend} attention backend: "
              + (f"{n_attn} of {f_attn} (sequence, KV-head) tree_attention units + " if f_attn else "")
              + f"target_dist/mss_verify of {n_acc} of {f_acc} sequences per step on a pool of {cores} "
              f"one-BLAS-thread processes" + ("" if full else ", scaled to the whole batch"))
    extra = {"sample_fraction": {"attention": (n_attn / f_attn) if f_attn else None, "accept": n_acc / f_acc},
             "pool_seconds_per_step": {"attention": attn_s * (n_attn / f_attn) if f_attn else 0.0,
                                       "accept": acc_s * n_acc / f_acc},
             "one_unit_seconds": {**{"attn_" + k: v for k, v in backends.items()}, "accept": one["accept"]}}
    return attn_s + acc_s, cores, sample, extra


def run_reference(args, cfg, mode):
    """--impl reference: the reference's own CPU implementation of the path
    (stock specdec from baseline/_ref, ``reference_pool``; the numpy oracle
    port when it is not installed), rank 0 only, every host core."""
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    port = None
    try:
        res = reference_pool(cfg, mode, args.steps, args.warmup)
    except Exception as e:  # noqa: BLE001 - report the port instead of failing the arm
        print(f"[bench] stock reference failed ({e!r}); timing the numpy port", file=sys.stderr)
        res = None
    if res is not None:
        step_s, cores, sample, extra = res
        kind = "reference"
        # the numpy port (oracle restatement) as a secondary figure
        ta, tacc, fa, facc = cpu_sample(cfg, seed=1, mode=mode)
        port = (ta * fa + tacc * facc) * 1e6
    else:
        cores = blas_threads()
        samples = []
        for i in range(args.warmup + args.steps):
            ta, tacc, fa, facc = cpu_sample(cfg, seed=i, mode=mode)
            if i >= args.warmup:
                samples.append(ta * fa + tacc * facc)
        step_s = statistics.mean(samples)
        kind = "port"
        sample = _sample_desc(cfg, mode, cores)
        extra = {}
    us = step_s * 1e6
    line = {"impl": "reference", "metric": METRIC, "value": us, "unit": "us/step", "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": step_s * 1e3, "higher_is_better": False,
            "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": cfg["workload"], "global_batch": cfg["B"], "seq_len": cfg["ctx"], "mode": mode},
            "cpu_baseline": {"value": us, "unit": "us/step", "cores": cores, "kind": kind, "sample": sample, **extra},
            "e2e": {"value": us, "unit": "us/step", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    if port is not None:
        line["cpu_baseline"]["port_us_per_step"] = port
    print(json.dumps(line), flush=True)


def graph_kernels(graph):
    """(this library's kernels, all kernels) among the kernel nodes of a
    captured step, by kernel name (namespace sdb), or None when the graph
    cannot be inspected."""
    try:
        from cuda.bindings import driver as cu

        g = cu.CUgraph(graph.raw_cuda_graph())
        err, _, n = cu.cuGraphGetNodes(g, 0)
        err, nodes, n = cu.cuGraphGetNodes(g, n)
        ours = total = 0
        others = []
        for nd in nodes[:n]:
            err, t = cu.cuGraphNodeGetType(nd)
            if t != cu.CUgraphNodeType.CU_GRAPH_NODE_TYPE_KERNEL:
                continue
            total += 1
            err, prm = cu.cuGraphKernelNodeGetParams(nd)
            err, name = cu.cuFuncGetName(prm.func)
            if err == cu.CUresult.CUDA_SUCCESS and b"sdb" in bytes(name):
                ours += 1
            else:
                others.append(bytes(name)[:60].decode(errors="replace"))
        if others:
            print(f"[bench] step graph: other kernels {others}", file=sys.stderr)
        return ours, total
    except Exception as e:  # noqa: BLE001 - diagnostic only
        print(f"[bench] graph inspection failed: {e}", file=sys.stderr)
        return None


def graph_time(fn, iters, stream, use_graph=True):
    """Mean device time of fn(): captured into a CUDA graph and replayed
    `iters` times between two events (host launch gaps excluded); eager
    launches when capture is not possible (gloo collectives)."""
    import torch

    g = None
    if use_graph:
        s = torch.cuda.Stream()
        s.wait_stream(stream)
        with torch.cuda.stream(s):
            fn()
        stream.wait_stream(s)
        torch.cuda.synchronize()
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g):
            fn()
        torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for _ in range(iters):
        g.replay() if g is not None else fn()
    e1.record(stream)
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / iters


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=50)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="c3", choices=sorted(CONFIGS))
    ap.add_argument("--mode", default=None, choices=["greedy", "stochastic"],
                    help="acceptance mode (default: greedy, c5: stochastic)")
    ap.add_argument("--kernel", type=int, default=0, help="0 auto, 1 tcgen05, 2 SIMT")
    ap.add_argument("--tree", default="64", choices=sorted(TREES),
                    help="64 / 65: R = 64 / 65 tree rows (63 / 64 drafts + root); chain3 / n8: the HBM-bound "
                         "contrast trees (R = 4 / 9)")
    ap.add_argument("--splits", type=int, default=0)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3)
    global TREE
    TREE = TREES[args.tree]
    cfg = dict(CONFIGS[args.config])
    if args.tree != "64":
        cfg["workload"] = cfg["workload"].replace("tree64", {"65": "tree65"}.get(args.tree, f"tree-{args.tree}"))
    mode = args.mode or cfg.get("mode", "greedy")
    accept_only = bool(cfg.get("accept_only"))
    if mode != "greedy" and not accept_only:
        cfg["workload"] = cfg["workload"].replace("greedy", f"stochastic T{TEMPERATURE:g} top-p {TOP_P:g}")
    if args.impl == "reference":
        run_reference(args, cfg, mode)
        return

    import numpy as np
    import torch
    import torch.distributed as dist

    from paper_2508_08192_b200 import _lib
    from paper_2508_08192_b200.kvstore import compact_kv
    from paper_2508_08192_b200.sharding import ShardedGreedyAcceptor, ShardedStochasticAcceptor, shard_for
    from paper_2508_08192_b200.verify import TreeVerifier

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    # SDB_BENCH_BACKEND=gloo exercises the sharded multi-rank path on a
    # one-GPU box (ranks share cuda:0); the product path is NCCL.
    backend = os.environ.get("SDB_BENCH_BACKEND", "nccl")
    local = local % max(1, torch.cuda.device_count())
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        if backend == "nccl":
            dist.init_process_group("nccl", device_id=dev)
        else:
            dist.init_process_group(backend)
    _lib.load()
    shard = shard_for(rank, world, cfg["Hq"], cfg["Hkv"], cfg["V"])
    x, R = make_inputs(cfg, shard, dev, mode=mode)
    aug = tuple(_augment(TREE))
    anc_pairs = _ancestor_pairs(aug)  # visible (row, tree key) pairs: the suffix part of the FLOP count
    n_parent_rows = len(set(p for p in aug[1:]))
    temperature = 0.0 if mode == "greedy" else TEMPERATURE
    ver = TreeVerifier(scale=cfg["d"] ** -0.5, temperature=temperature, top_p=TOP_P if mode != "greedy" else 1.0,
                       max_ctx=max(cfg["ctx"], 1), num_splits=args.splits, kernel=args.kernel,
                       reserve_sms=(int(os.environ["SDB_RESERVE_SMS"]) if "SDB_RESERVE_SMS" in os.environ else None),
                       tree_levels=_tree_levels(aug))
    if os.environ.get("SDB_STOCH_EAGER"):  # A/B: reduce every row (no lazy walk)
        ver.stochastic.lazy = False
    if world > 1:
        if mode == "greedy":
            sharded = ShardedGreedyAcceptor(shard)
            ver.greedy = lambda logits, parent, n_rows, tokens, stream=None: sharded(logits, parent, n_rows, tokens,
                                                                                    stream)
        else:
            nch = max(sum(1 for q in aug if q == p_) for p_ in set(aug[1:]))
            ver.stochastic = ShardedStochasticAcceptor(shard, max_children=nch)
    stream = torch.cuda.current_stream()
    o = ver._buffers(x)

    def part_build():
        lib = _lib.lib()
        b_, r_ = x.parent.shape
        _lib.check(lib.sdb_tree_build(_lib.ptr(x.parent), _lib.ptr(x.n_rows), _lib.ptr(x.ctx_len), b_, r_,
                                      o["mask"].shape[-1], _lib.ptr(o["mask"]), _lib.ptr(o["pos"]),
                                      _lib.ptr(o["depth"]), _lib.ptr(o["tree_err"]), _lib.stream_ptr()), "tree_build")

    def part_attn():
        ver.attn(x.q, x.k_pool, x.v_pool, x.block_table, x.ctx_len, x.tree_k, x.tree_v, o["mask"], x.n_rows,
                 ver.scale, out=o["out"], lse=o["lse"], max_ctx=ver.max_ctx, num_splits=ver.num_splits,
                 kernel=ver.kernel)

    acc_box = {}

    def part_accept():
        if mode == "greedy":
            acc_box["acc"] = ver.greedy(x.logits, x.parent, x.n_rows, x.tokens)
        else:
            acc_box["acc"] = ver.stochastic(x.logits, x.draft_logits, temperature, TOP_P, x.parent, x.n_rows,
                                            x.tokens, None, seeds=x.seeds, steps=x.steps)

    def part_compact():
        acc = acc_box["acc"]
        compact_kv(x.tree_k.unsqueeze(0), x.tree_v.unsqueeze(0), x.k_pool.unsqueeze(0), x.v_pool.unsqueeze(0),
                   x.block_table, x.ctx_len, acc.path, acc.path_len)

    if accept_only:
        def step():
            part_accept()
    else:
        def step():
            return ver.step(x)

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    # CUDA graph of the whole step (NCCL collectives included for N > 1: the
    # communicator is warm after the eager warm-up steps); gloo cannot be
    # captured and runs eagerly.
    use_graph = world == 1 or backend == "nccl"
    graph = None
    if use_graph:
        try:
            s_ = torch.cuda.Stream()
            s_.wait_stream(stream)
            with torch.cuda.stream(s_):
                step()
            stream.wait_stream(s_)
            torch.cuda.synchronize()
            graph = torch.cuda.CUDAGraph()
            with torch.cuda.graph(graph):
                step()
        except Exception as e:  # noqa: BLE001 - fall back to eager steps, reported in config.graph
            print(f"[bench] rank {rank}: graph capture failed ({e}); timing eager steps", file=sys.stderr)
            use_graph, graph = False, None
            torch.cuda.synchronize()
        if world > 1:  # every rank times the same mode
            ok = torch.tensor([1 if use_graph else 0], dtype=torch.int32, device=dev)
            dist.all_reduce(ok, op=dist.ReduceOp.MIN)
            use_graph = bool(ok.item())
    torch.cuda.synchronize()

    def barrier():
        if world > 1:
            dist.barrier()

    # ---- timed region: K steps, device events, max over ranks ----------
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    sampler = ClockSampler(local)
    barrier()
    torch.cuda.synchronize()
    with sampler:
        e0.record(stream)
        for _ in range(args.steps):
            if use_graph:
                graph.replay()
            else:
                step()
        e1.record(stream)
        torch.cuda.synchronize()
    barrier()
    ms = e0.elapsed_time(e1) / args.steps
    t = torch.tensor([ms], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    ms = float(t.item())

    # ---- per-kernel breakdown: each part graph-replayed alone ------------
    barrier()
    parts = {}
    if not accept_only:
        parts["tree_build"] = graph_time(part_build, args.steps, stream, use_graph)
        parts["tree_attn"] = graph_time(part_attn, args.steps, stream, use_graph)
    parts["accept"] = graph_time(part_accept, args.steps, stream, use_graph)
    if not accept_only:
        parts["compact"] = graph_time(part_compact, args.steps, stream, use_graph)
    acc = acc_box["acc"]
    accept_len = float(acc.path_len.float().mean().item())

    # ---- e2e through the public API with host buffers ----------------------
    e2e = None
    if not args.no_e2e:
        names = ["logits", "parent", "n_rows", "ctx_len", "tokens"]
        if not accept_only:
            names += ["q", "tree_k", "tree_v"]
        if mode != "greedy":
            names += ["draft_logits", "seeds", "steps"]
        pinned = {k: getattr(x, k).cpu().pin_memory() for k in names}
        dev_in = {k: torch.empty_like(getattr(x, k)) for k in pinned}
        h2d = sum(v.numel() * v.element_size() for v in pinned.values())
        host_out = {"path": acc.path, "path_len": acc.path_len, "next_token": acc.next_token}
        if not accept_only:
            host_out.update(out=o["out"], lse=o["lse"])
        outs_h = {k: torch.empty(v.shape, dtype=v.dtype).pin_memory() for k, v in host_out.items()}
        d2h = sum(t_.numel() * t_.element_size() for t_ in outs_h.values())
        from paper_2508_08192_b200.verify import StepInputs

        fields = {k: getattr(x, k) for k in StepInputs.__dataclass_fields__}
        fields.update(dev_in)
        xe = StepInputs(**fields)

        # full step: host inputs -> host outputs through the public pipelined
        # API (chunks of sequences: H2D of chunk c+1 under the step of chunk c)
        e2e_chunks = int(os.environ.get("SDB_E2E_CHUNKS", "4"))
        pipe = None
        if not accept_only and e2e_chunks > 1 and world == 1:
            from paper_2508_08192_b200.verify import HostStepPipeline

            def make_chunk_verifier():
                v_ = TreeVerifier(scale=ver.scale, temperature=ver.temperature, top_p=ver.top_p,
                                  max_ctx=ver.max_ctx, num_splits=ver.num_splits, kernel=ver.kernel,
                                  reserve_sms=ver.reserve_sms, tree_levels=ver.stochastic.levels)
                v_.stochastic.lazy = ver.stochastic.lazy
                return v_

            pipe = HostStepPipeline(make_chunk_verifier, chunks=e2e_chunks)

        def e2e_step():
            if pipe is not None:
                pipe(xe, pinned, outs_h, stream)
                return
            for k_, v_ in pinned.items():
                dev_in[k_].copy_(v_, non_blocking=True)
            if accept_only:
                ver_acc = (ver.greedy(xe.logits, xe.parent, xe.n_rows, xe.tokens) if mode == "greedy" else
                           ver.stochastic(xe.logits, xe.draft_logits, temperature, TOP_P, xe.parent, xe.n_rows,
                                          xe.tokens, None, seeds=xe.seeds, steps=xe.steps))
                res = {"path": ver_acc.path, "path_len": ver_acc.path_len, "next_token": ver_acc.next_token}
            else:
                out_, lse_, acc_, _ = ver.step(xe)
                res = {"path": acc_.path, "path_len": acc_.path_len, "next_token": acc_.next_token, "out": out_,
                       "lse": lse_}
            for k_, v_ in res.items():
                outs_h[k_].copy_(v_, non_blocking=True)

        for _ in range(2):
            e2e_step()
        torch.cuda.synchronize()
        barrier()
        f0, f1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        f0.record(stream)
        for _ in range(args.steps):
            e2e_step()
        f1.record(stream)
        torch.cuda.synchronize()
        e2e_ms = f0.elapsed_time(f1) / args.steps
        te = torch.tensor([e2e_ms], dtype=torch.float64, device=dev)
        if world > 1:
            dist.all_reduce(te, op=dist.ReduceOp.MAX)
        e2e = {"value": float(te.item()) * 1e3, "unit": "us/step", "h2d_bytes_per_step": int(h2d),
               "d2h_bytes_per_step": int(d2h), "chunks": e2e_chunks if pipe is not None else 1}
        # the host outputs of the last e2e step equal the device step's (same inputs)
        e2e["parity"] = bool(torch.equal(outs_h["path_len"], acc.path_len.cpu())
                             and torch.equal(outs_h["next_token"], acc.next_token.cpu())
                             and all(torch.equal(outs_h["path"][b_, :int(acc.path_len[b_])],
                                                 acc.path[b_, :int(acc.path_len[b_])].cpu())
                                     for b_ in range(acc.path_len.shape[0])))

    attn_bytes, accept_bytes, attn_flops = step_bytes_flops(cfg, shard, R, anc_pairs)
    if mode != "greedy":
        # target rows + the draft rows that carry a q (parents), SURVEY 8(d)
        accept_bytes = cfg["B"] * (R + n_parent_rows) * shard.n_vocab * 4
    if accept_only:
        attn_bytes, attn_flops = 0, 0.0
    tot = torch.tensor([attn_bytes + accept_bytes], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(tot)
    step_bytes_all = float(tot.item())
    hbm_peak, tc_peak, peak_src = _measured_peaks()
    traffic = None
    try:
        with open(os.path.join(ROOT, "profiles", "attn_traffic.json")) as f:
            traffic = json.load(f).get(f"{args.config}:{mode}:g{world}" + ("" if args.tree == "64" else f":{args.tree}"))
    except Exception:
        pass
    gbs = step_bytes_all / (ms * 1e-3) / 1e9
    t_acc = parts["accept"]
    accept_gbs = accept_bytes / (t_acc * 1e-3) / 1e9
    if accept_only:
        roof = {"kernel": "accept_" + mode, "bound": "hbm", "achieved": accept_gbs, "peak": hbm_peak,
                "unit": "GB/s", "frac": accept_gbs / hbm_peak, "traffic": traffic, "peak_source": peak_src,
                "bytes_per_launch": accept_bytes}
    else:
        t_attn_ms = parts["tree_attn"]
        achieved_tf = attn_flops / (t_attn_ms * 1e-3) / 1e12
        attn_gbs = attn_bytes / (t_attn_ms * 1e-3) / 1e9
        # the binding bound of the attention: tensor at C3/C4, HBM at bs 1 (C2)
        if attn_bytes / (hbm_peak * 1e9) > attn_flops / (tc_peak * 1e12):
            roof = {"kernel": "tree_attn", "bound": "hbm", "achieved": attn_gbs, "peak": hbm_peak, "unit": "GB/s",
                    "frac": attn_gbs / hbm_peak, "traffic": traffic, "peak_source": peak_src,
                    "bytes_per_launch": attn_bytes, "tflops": achieved_tf,
                    "accept_hbm_gbs": accept_gbs, "accept_hbm_frac": accept_gbs / hbm_peak}
        else:
            roof = {"kernel": "tree_attn", "bound": "tensor", "achieved": achieved_tf, "peak": tc_peak,
                    "unit": "TFLOP/s", "frac": achieved_tf / tc_peak, "traffic": traffic, "peak_source": peak_src,
                    "flops_per_launch": attn_flops, "hbm_gbs": attn_gbs,
                    "accept_hbm_gbs": accept_gbs, "accept_hbm_frac": accept_gbs / hbm_peak}
    # step-level roofline: the attention's binding bound (tensor at C3/C4)
    # plus the acceptance's HBM bound, executed back to back
    t_attn_star = 0.0 if accept_only else max(attn_flops / (tc_peak * 1e12), attn_bytes / (hbm_peak * 1e9))
    t_star = t_attn_star + accept_bytes / (hbm_peak * 1e9)
    step_roof = {"t_star_us": t_star * 1e6, "frac": t_star / (ms * 1e-3),
                 "how": "max(attention FLOPs / measured bf16 peak, attention bytes / measured HBM) + acceptance "
                        "bytes / measured HBM"}
    # library kernels per step: tree_build 1, attention 2 (persistent kernel +
    # LSE fix-up), acceptance 2 (greedy: keys + walk; stochastic: row stats +
    # walk, + 1 Philox), compaction 1
    # our kernels per step: counted from the captured graph's kernel nodes;
    # eager (gloo) runs fall back to the static count of the step's launches
    n_launch = (0 if accept_only else 4) + (2 if mode == "greedy" else 3)
    counted = None
    if graph is not None:
        # a second, kept capture of the step only to count its kernel nodes
        # (the timed graph is not kept: keep_graph=True measured +4 us at C2)
        try:
            kept = torch.cuda.CUDAGraph(keep_graph=True)
            with torch.cuda.graph(kept):
                step()
            counted = graph_kernels(kept)
            del kept
        except Exception as e:  # noqa: BLE001 - diagnostic only
            print(f"[bench] kernel count capture failed: {e}", file=sys.stderr)
        torch.cuda.synchronize()
    if counted is not None:
        n_launch = counted[0]
        if counted[1] != counted[0]:
            print(f"[bench] step graph: {counted[0]} library kernels of {counted[1]}", file=sys.stderr)
    line = {
        "metric": METRIC, "value": ms * 1e3, "unit": "us/step", "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": False, "scaling": "strong",
        "vs_baseline": None, "dtype": "bf16" if not accept_only else "f32", "data": "synthetic",
        "config": {"workload": cfg["workload"], "global_batch": cfg["B"], "seq_len": cfg["ctx"], "tree_rows": R,
                   "heads": f"{cfg['Hq']}q/{cfg['Hkv']}kv d{cfg['d']}", "page": cfg["bs"], "vocab": cfg["V"],
                   "mode": mode, "parallelism": f"kv-head+vocab shard x{world}",
                   "l2": f"inputs {(attn_bytes + accept_bytes) / 1e9:.1f} GB/GPU >> 126 MB L2", "graph": use_graph},
        "hbm_gbs": gbs, "pct_of_8tbs": 100.0 * gbs / 8000.0,
        "kernels_ms": parts,
        "mean_accepted": accept_len,
        "roofline": roof,
        "step_roofline": step_roof,
        "clocks": sampler.summary(),
        "gpu_launches": n_launch * args.steps,
        "e2e": e2e,
    }
    parity = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        # the oracle leg: one sampled sequence of the measured outputs checked ...
        parity = parity_sample(cfg, x, None if accept_only else o["out"], None if accept_only else o["lse"], acc,
                               mode, aug)
        line["parity"] = parity
        # ... and the reference timed on the host: the stock path on every
        # core for two steps (the same measurement as --impl reference;
        # spawned workers: this process holds a CUDA context), else the port
        try:
            res = reference_pool(cfg, mode, steps=2, warmup=1, start="spawn")
        except Exception as e:  # noqa: BLE001 - the reference is optional here: fall back to the port
            print(f"[bench] stock reference timing failed ({e!r}); timing the numpy port", file=sys.stderr)
            res = None
        if res is not None:
            step_s, cores, sample, extra = res
            line["cpu_baseline"] = {"value": step_s * 1e6, "unit": "us/step", "cores": cores, "kind": "reference",
                                    "sample": sample, **extra}
        else:
            cpu_sample(cfg, mode=mode)
            ta, tacc, fa, facc = cpu_sample(cfg, seed=1, mode=mode)
            us = (ta * fa + tacc * facc) * 1e6
            line["cpu_baseline"] = {"value": us, "unit": "us/step", "cores": blas_threads(), "kind": "port",
                                    "sample": _sample_desc(cfg, mode, blas_threads())}
    if rank == 0:
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()
    if parity is not None and not parity["ok"]:
        print(f"[bench] PARITY FAILURE vs the oracle: {parity}", file=sys.stderr)
        sys.exit(1)


if __name__ == "__main__":
    main()
