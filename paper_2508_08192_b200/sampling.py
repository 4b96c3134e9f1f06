"""Target distributions and tree acceptance on the GPU.

Drop-in layer (numpy float64 in/out, reference names and errors,
sampling.py:23-202): ``target_dist``, ``top_p_mask``, ``sample_from``,
``mss_verify`` run float64 kernels (sdb_target_dist_f64, sdb_mss_verify_f64).
``rank_sliced_uniforms`` stays a host function exactly as in the reference
(the uniforms are an *input* of the path; a device Philox is SURVEY.md
section 8f row 3).

Perf layer: ``accept_greedy`` (T = 0: packed-key argmax + tree walk) and
``accept_stochastic`` (T > 0: nucleus stats + MSS walk) over batched fp32 /
bf16 logits on the device.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from . import _lib
from .drafttree import TreeSpec


class SamplingError(ValueError):
    pass


@dataclass(frozen=True)
class SamplerConfig:
    temperature: float = 1.0
    top_p: float = 1.0
    seed: int = 0
    simulated_world_size: int = 1

    def __post_init__(self):
        if self.temperature < 0:
            raise SamplingError("temperature must be >= 0")
        if not 0 < self.top_p <= 1:
            raise SamplingError("top_p must be in (0, 1]")
        if self.simulated_world_size < 1:
            raise SamplingError("simulated_world_size must be >= 1")


def check_dist(dist):
    """sampling.py:43-49 (host-side argument validation)."""
    d = np.asarray(dist, dtype=np.float64)
    if d.ndim != 1:
        raise SamplingError(f"distribution must be 1-D, got {d.shape}")
    if (d < 0).any() or abs(float(d.sum()) - 1.0) > 1e-9:
        raise SamplingError("distribution entries must be >= 0 and sum to 1")
    return d


def _dev(x, dtype=np.float64):
    import torch

    return torch.from_numpy(np.ascontiguousarray(x, dtype=dtype)).cuda()


def _raise_err(code, what):
    if code & _lib.SDB_ERR_NAN:
        raise ValueError(f"{what}: NaN in logits")
    if code & _lib.SDB_ERR_NO_ALLOWED:
        raise SamplingError("no token allowed (dead FSM state)")
    if code & _lib.SDB_ERR_BAD_DIST:
        raise SamplingError("distribution entries must be >= 0 and sum to 1")
    if code & _lib.SDB_ERR_UNIFORMS:
        raise SamplingError("uniform stream exhausted")
    if code & _lib.SDB_ERR_PLAN:
        raise SamplingError("tree deeper / wider than the planned walk levels")
    if code & _lib.SDB_ERR_CACHE:
        from .kvstore import CacheError

        raise CacheError("write past allocated blocks")


def target_dists(logits, temperature, top_p, allowed=None):
    """Batched drop-in: logits (rows, V) -> distributions (rows, V) float64."""
    import torch

    lg = np.atleast_2d(np.asarray(logits, dtype=np.float64))
    rows, vocab = lg.shape
    if temperature < 0:
        raise ValueError("softmax_lse: negative temperature")
    if not 0 < top_p <= 1:
        raise SamplingError("top_p must be in (0, 1]")
    al = None
    if allowed is not None:
        al = _dev(np.broadcast_to(np.asarray(allowed, dtype=bool), lg.shape), np.uint8)
    tl = _dev(lg)
    out = torch.empty_like(tl)
    err = torch.zeros((1,), dtype=torch.int32, device="cuda")
    rc = _lib.lib().sdb_target_dist_f64(_lib.ptr(tl), _lib.ptr(al), rows, vocab, float(temperature),
                                        float(top_p), _lib.ptr(out), _lib.ptr(err), _lib.stream_ptr())
    _lib.check(rc, "target_dist")
    _raise_err(int(err.item()), "softmax_lse")
    return out.cpu().numpy()


def target_dist(logits_row, temperature, top_p, allowed=None):
    """Logits row -> sampling distribution: mask, temperature, top-p
    (sampling.py:87-102)."""
    row = np.asarray(logits_row, dtype=np.float64)
    if allowed is not None and not np.asarray(allowed).any():
        raise SamplingError("no token allowed (dead FSM state)")
    return target_dists(row[None, :], temperature, top_p, None if allowed is None else allowed[None, :])[0]


def top_p_mask(dist, p):
    """sampling.py:57-72 on the device: the nucleus of a distribution is the
    nucleus of its logits at T = 1 (log is monotone, softmax(log d) = d)."""
    d = check_dist(dist)
    if not 0 < p <= 1:
        raise SamplingError("top_p must be in (0, 1]")
    with np.errstate(divide="ignore"):
        lg = np.log(d)
    return target_dists(lg[None, :], 1.0, p)[0]


def greedy_expand(dist, k):
    """Top-k tokens by probability, lowest index on ties (sampling.py:75-84).
    Drafting-side helper, host only."""
    d = check_dist(dist)
    if not 1 <= k <= d.shape[0]:
        raise SamplingError(f"k={k} out of range for vocab {d.shape[0]}")
    return [int(t) for t in np.lexsort((np.arange(d.shape[0]), -d))[:k]]


def rank_sliced_uniforms(seed, step, padded_batch, row_width):
    """Philox uniforms keyed by (seed, step) (sampling.py:112-124)."""
    if padded_batch < 1 or row_width < 0:
        raise SamplingError("padded_batch must be >= 1 and row_width >= 0")
    key = np.array([np.uint64(seed & 0xFFFFFFFFFFFFFFFF), np.uint64(step & 0xFFFFFFFFFFFFFFFF)], dtype=np.uint64)
    gen = np.random.Generator(np.random.Philox(key=key))
    return gen.random((padded_batch, row_width), dtype=np.float64)


@dataclass
class DraftResult:
    tree: TreeSpec
    node_tokens: tuple
    node_dists: tuple


@dataclass
class MssResult:
    accepted_path: list
    next_token: int
    residual: np.ndarray
    uniforms_used: int


def mss_verify(draft, target_dists_, uniforms, mode="greedy_children"):
    """Multi-round speculative sampling on the device (sampling.py:149-202)."""
    import torch

    if mode not in ("stochastic", "greedy_children"):
        raise SamplingError(f"unknown mss mode {mode!r}")
    tree = draft.tree
    n = tree.n_nodes
    if len(target_dists_) != n + 1:
        raise SamplingError("need one target dist per node parent incl. root")
    td = np.stack([np.asarray(d, dtype=np.float64) for d in target_dists_])
    vocab = td.shape[1]
    if td.ndim != 2:
        raise SamplingError("distribution must be 1-D")
    uni = np.asarray(uniforms, dtype=np.float64).reshape(-1)
    nd = np.stack([np.asarray(d, dtype=np.float64) for d in draft.node_dists]) if n else np.zeros((1, vocab))
    par = _dev(np.asarray(tree.parent if n else [-1]), np.int32)
    tok = _dev(np.asarray(draft.node_tokens if n else [0]), np.int32)
    path = torch.zeros((max(n, 1),), dtype=torch.int32, device="cuda")
    scal = torch.zeros((3,), dtype=torch.int64, device="cuda")
    resid = torch.empty((vocab,), dtype=torch.float64, device="cuda")
    err = torch.zeros((1,), dtype=torch.int32, device="cuda")
    tu = _dev(uni if uni.size else np.zeros(1))
    tnd, ttd = _dev(nd), _dev(td)  # keep alive until the launch is enqueued
    rc = _lib.lib().sdb_mss_verify_f64(_lib.ptr(par), _lib.ptr(tok), n, vocab, _lib.ptr(tnd),
                                       _lib.ptr(ttd), _lib.ptr(tu), int(uni.size), _lib.ptr(path),
                                       _lib.ptr(scal), _lib.ptr(resid), _lib.ptr(err), _lib.stream_ptr())
    _lib.check(rc, "mss_verify")
    e = int(err.item())
    if e & _lib.SDB_ERR_BAD_DIST:
        raise SamplingError("distribution entries must be >= 0 and sum to 1")
    if e & _lib.SDB_ERR_UNIFORMS:
        raise SamplingError("uniform stream exhausted")
    s = scal.cpu().numpy()
    plen = int(s[0])
    return MssResult([int(x) for x in path[:plen].cpu().numpy()], int(s[1]), resid.cpu().numpy(), int(s[2]))


def sample_from(dist, u):
    """Inverse-CDF draw (sampling.py:105-109): the bonus draw of an empty-tree
    mss_verify on the device."""
    d = check_dist(dist)
    res = mss_verify(DraftResult(TreeSpec(()), (), ()), [d], [u])
    return res.next_token


# ---------------------------------------------------------------------------
# batched device acceptance
# ---------------------------------------------------------------------------

@dataclass
class AcceptResult:
    path: "object"           # int32 [B, R] draft-node indices (first path_len valid)
    path_len: "object"       # int32 [B]
    next_token: "object"     # int64 [B]
    uniforms_used: "object"  # int32 [B]
    err: "object"            # int32 [1] device error bits
    residual: "object" = None

    def raise_if_error(self, what="acceptance"):
        """Host sync: map the device error bits to the reference exceptions
        (ValueError for NaN, SamplingError, CacheError for a compaction
        past the mapped blocks)."""
        if self.err is not None:
            _raise_err(int(self.err.reshape(-1)[0].item()), what)


class GreedyAcceptor:
    """T = 0 acceptance with preallocated outputs (graph-capturable)."""

    def __init__(self):
        self._bufs = None

    def _alloc(self, b, r, dev):
        import torch

        key = (b, r, str(dev))
        if self._bufs is None or self._bufs[0] != key:
            self._bufs = (key, dict(
                keys=torch.empty((b, r, 8), dtype=torch.int64, device=dev),  # SDB_GREEDY_KEY_SLOTS
                path=torch.zeros((b, r), dtype=torch.int32, device=dev),
                path_len=torch.empty((b,), dtype=torch.int32, device=dev),
                next_token=torch.empty((b,), dtype=torch.int64, device=dev),
                used=torch.empty((b,), dtype=torch.int32, device=dev),
                err=torch.zeros((1,), dtype=torch.int32, device=dev)))
        return self._bufs[1]

    def __call__(self, logits, parent, n_rows, tokens, stream=None, allowed=None):
        import torch

        b, r, v = logits.shape
        if allowed is not None:
            return self._masked(logits, parent, n_rows, tokens, allowed, stream)
        if logits.dtype == torch.float32:
            dt = _lib.DTYPE_F32
        elif logits.dtype == torch.bfloat16:
            dt = _lib.DTYPE_BF16
        else:
            raise SamplingError(f"unsupported logits dtype {logits.dtype}")
        if logits.is_contiguous():
            row_stride = v
        elif logits.stride(2) == 1 and (b == 1 or logits.stride(0) == r * logits.stride(1)):
            row_stride = logits.stride(1)
        else:
            raise SamplingError("logits must be [B, R, V] with unit vocab stride and uniform row stride")
        o = self._alloc(b, r, logits.device)
        _lib.clear(o["err"], stream)
        rc = _lib.lib().sdb_accept_greedy(_lib.ptr(logits), dt, b, r, v, row_stride, _lib.ptr(parent),
                                          _lib.ptr(n_rows), _lib.ptr(tokens), _lib.ptr(o["keys"]),
                                          _lib.ptr(o["path"]), _lib.ptr(o["path_len"]), _lib.ptr(o["next_token"]),
                                          _lib.ptr(o["used"]), _lib.ptr(o["err"]), _lib.stream_ptr(stream))
        _lib.check(rc, "accept_greedy")
        return AcceptResult(o["path"], o["path_len"], o["next_token"], o["used"], o["err"])


    def _masked(self, logits, parent, n_rows, tokens, allowed, stream):
        import torch

        b, r, v = logits.shape
        if logits.dtype != torch.float32 or logits.stride(2) != 1 or allowed.dtype != torch.int32:
            raise SamplingError("masked greedy acceptance takes fp32 logits and int32 allowed words")
        o = self._alloc(b, r, logits.device)
        _lib.clear(o["err"], stream)
        rc = _lib.lib().sdb_accept_greedy_ex(_lib.ptr(logits), b, r, v, logits.stride(1), _lib.ptr(parent),
                                             _lib.ptr(n_rows), _lib.ptr(tokens), _lib.ptr(allowed), allowed.shape[-1],
                                             _lib.ptr(o["keys"]), _lib.ptr(o["path"]), _lib.ptr(o["path_len"]),
                                             _lib.ptr(o["next_token"]), _lib.ptr(o["used"]), _lib.ptr(o["err"]),
                                             _lib.stream_ptr(stream))
        _lib.check(rc, "accept_greedy_ex")
        return AcceptResult(o["path"], o["path_len"], o["next_token"], o["used"], o["err"])

    def fused_keys(self, b, r, dev):
        """Key buffer + error word for the attention-fused argmax scan."""
        o = self._alloc(b, r, dev)
        return o["keys"], o["err"]

    def walk(self, parent, n_rows, tokens, stream=None):
        """The greedy walk on keys produced by the attention-fused scan
        (sdb_tree_attn fused_keys); err was zeroed by the caller."""
        b, r = parent.shape
        o = self._alloc(b, r, parent.device)
        rc = _lib.lib().sdb_greedy_walk(_lib.ptr(o["keys"]), _lib.ptr(parent), _lib.ptr(n_rows), _lib.ptr(tokens),
                                        b, r, _lib.ptr(o["path"]), _lib.ptr(o["path_len"]),
                                        _lib.ptr(o["next_token"]), _lib.ptr(o["used"]), _lib.stream_ptr(stream))
        _lib.check(rc, "greedy_walk")
        return AcceptResult(o["path"], o["path_len"], o["next_token"], o["used"], o["err"])


def pack_allowed(mask):
    """bool [..., V] allowed-token mask -> int32 words [..., ceil(V / 32)]
    (bit j of word w = token 32 w + j), the layout of the masked acceptance."""
    import torch

    v = mask.shape[-1]
    w = -(-v // 32)
    pad = torch.zeros(mask.shape[:-1] + (w * 32,), dtype=torch.int64, device=mask.device)
    pad[..., :v] = mask.to(torch.int64)
    bits = pad.reshape(mask.shape[:-1] + (w, 32)) << torch.arange(32, device=mask.device, dtype=torch.int64)
    words = bits.sum(-1)
    return torch.where(words >= 2**31, words - 2**32, words).to(torch.int32)


def accept_greedy(logits, parent, n_rows, tokens, stream=None, allowed=None):
    """Batched temperature-0 acceptance.

    logits [B, R, V] fp32/bf16 (row r = augmented tree row r); parent int32
    [B, R] augmented (row 0 = root, parent -1); tokens int32 [B, R] (token of
    row r, row 0 ignored); n_rows int32 [B].  Returns device tensors; no host
    synchronisation.  ``allowed``: int32 words from ``pack_allowed`` (FSM
    masks per row, guided decoding) or None."""
    return GreedyAcceptor()(logits, parent, n_rows, tokens, stream, allowed)


def argmax_keys(logits2d, vocab_offset=0, stream=None):
    """Packed int64 argmax keys of a (rows, V_local) logits shard (vocab
    shard starting at vocab_offset); all-reduce MAX across shards gives the
    global argmax with the lowest index on ties."""
    import torch

    rows, v = logits2d.shape
    dt = _lib.DTYPE_F32 if logits2d.dtype == torch.float32 else _lib.DTYPE_BF16
    keys = torch.empty((rows,), dtype=torch.int64, device=logits2d.device)
    err = torch.zeros((1,), dtype=torch.int32, device=logits2d.device)
    rc = _lib.lib().sdb_argmax_keys(_lib.ptr(logits2d), dt, rows, v, logits2d.stride(0), int(vocab_offset),
                                    _lib.ptr(keys), _lib.ptr(err), _lib.stream_ptr(stream))
    _lib.check(rc, "argmax_keys")
    return keys, err


def greedy_walk(keys, parent, n_rows, tokens, stream=None):
    import torch

    b, r = parent.shape
    dev = parent.device
    path = torch.zeros((b, r), dtype=torch.int32, device=dev)
    plen = torch.empty((b,), dtype=torch.int32, device=dev)
    nxt = torch.empty((b,), dtype=torch.int64, device=dev)
    used = torch.empty((b,), dtype=torch.int32, device=dev)
    rc = _lib.lib().sdb_greedy_walk(_lib.ptr(keys), _lib.ptr(parent), _lib.ptr(n_rows), _lib.ptr(tokens), b, r,
                                    _lib.ptr(path), _lib.ptr(plen), _lib.ptr(nxt), _lib.ptr(used),
                                    _lib.stream_ptr(stream))
    _lib.check(rc, "greedy_walk")
    return AcceptResult(path, plen, nxt, used, None)


def device_uniforms(seeds, steps, width, row=0, out=None, stream=None):
    """Per-sequence uniform rows on the device, bit-identical to
    ``rank_sliced_uniforms(seeds[b], steps[b], padded, width)[row]``
    (sampling.py:112-124; the engine takes row 0, engine.py:251-254).

    seeds/steps: int64 device tensors [B] (uint64 bit patterns).  Returns
    float64 [B, width]."""
    import torch

    if seeds.dtype != torch.int64 or steps.dtype != torch.int64 or seeds.shape != steps.shape or seeds.dim() != 1:
        raise SamplingError("seeds and steps must be int64 [B] device tensors")
    if width < 0 or row < 0:
        raise SamplingError("padded_batch must be >= 1 and row_width >= 0")
    b = seeds.shape[0]
    if out is None:
        out = torch.empty((b, width), dtype=torch.float64, device=seeds.device)
    rc = _lib.lib().sdb_philox_uniforms(_lib.ptr(seeds), _lib.ptr(steps), b, int(row), int(width), _lib.ptr(out),
                                        _lib.stream_ptr(stream))
    _lib.check(rc, "philox_uniforms")
    return out


def tree_levels(parent):
    """Max depth + 1 of augmented parent rows [B, R] (host sync)."""
    par = parent.cpu().numpy()
    best = 1
    for row in par:
        depth = [0] * len(row)
        for i, p in enumerate(row):
            depth[i] = 0 if p < 0 else depth[p] + 1
        best = max(best, max(depth) + 1)
    return best


# diagnostics only (timing the lazy walk alone): skips the every-row validation
_DIAG_SKIP_VALIDATE = bool(__import__("os").environ.get("SDB_DIAG_SKIP_VALIDATE"))


class StochasticAcceptor:
    """T > 0 acceptance with a cached workspace (graph-capturable).

    ``lazy``: only the rows the MSS walk visits are reduced, one tree level
    per launch pair, while a validation scan of every row (the reference's
    error behaviour) runs concurrently on a side stream (a persistent kernel on
    52 of 148 SMs; the chain takes the rest); "auto" picks it from 20
    sequences up.  ``levels`` (tree depth + 1) must be given when
    capturing a CUDA graph.  Results are identical either way."""

    def __init__(self, lazy="auto", levels=None):
        self._ws = None
        self._bufs = None
        self.lazy = lazy
        self.levels = levels
        self._side = None

    def __call__(self, target_logits, draft_logits, temperature, top_p, parent, n_rows, tokens, uniforms=None,
                 want_residual=False, stream=None, seeds=None, steps=None, allowed=None):
        import torch

        b, r, v = target_logits.shape
        if target_logits.dtype != torch.float32 or draft_logits.dtype != torch.float32:
            raise SamplingError("stochastic acceptance takes fp32 logits")
        # every stochastic kernel indexes rows as (b * r_max + r) * vocab
        if (not target_logits.is_contiguous() or not draft_logits.is_contiguous()
                or draft_logits.shape != target_logits.shape):
            raise SamplingError("stochastic acceptance takes contiguous [B, R, V] target and draft logits")
        if uniforms is not None and (uniforms.dtype != torch.float64 or uniforms.dim() != 2
                                     or uniforms.shape[0] != b or not uniforms.is_contiguous()):
            raise SamplingError("uniforms must be a contiguous float64 [B, n_uniforms] tensor")
        if not (temperature > 0):
            raise SamplingError("stochastic acceptance needs temperature > 0 (use accept_greedy)")
        dev = target_logits.device
        lib = _lib.lib()
        need = lib.sdb_accept_stochastic_workspace(b, r, v)
        if self._ws is None or self._ws.numel() < need or self._ws.device != dev:
            self._ws = torch.empty((int(need),), dtype=torch.uint8, device=dev)
        key = (b, r, v, str(dev), want_residual)
        if self._bufs is None or self._bufs[0] != key:
            self._bufs = (key, dict(
                path=torch.zeros((b, r), dtype=torch.int32, device=dev),
                path_len=torch.empty((b,), dtype=torch.int32, device=dev),
                next_token=torch.empty((b,), dtype=torch.int64, device=dev),
                used=torch.empty((b,), dtype=torch.int32, device=dev),
                err=torch.zeros((1,), dtype=torch.int32, device=dev),
                residual=torch.empty((b, v), dtype=torch.float32, device=dev) if want_residual else None))
        o = self._bufs[1]
        _lib.clear(o["err"], stream)
        if uniforms is None:
            # (seeds, steps) on the device: the Philox rows are generated in
            # a launch on the same stream (no host transfer of uniforms)
            if seeds is None or steps is None:
                raise SamplingError("pass uniforms, or seeds and steps")
            if "uni" not in o or o["uni"].shape != (b, r):
                o["uni"] = torch.empty((b, r), dtype=torch.float64, device=dev)
            uniforms = device_uniforms(seeds, steps, r, out=o["uni"], stream=stream)
        n_words = allowed.shape[-1] if allowed is not None else 0
        # the lazy walk + concurrent validation scan (persistent, on 52 of
        # 148 SMs) costs ~440 us at B 16-20 and grows slowly; reducing every
        # row costs ~20 us per sequence (tools/lazy_sweep.py, V 128k,
        # tree64): lazy wins from about 20 sequences (B 16: 387 eager / 436
        # lazy; B 20: 462 / 449; B 32: 688 / 491; B 64: 1321 / 620 us)
        lazy = self.lazy if self.lazy != "auto" else (b >= 20)
        levels = self.levels
        if lazy and levels is None and not torch.cuda.is_current_stream_capturing():
            levels = tree_levels(parent)
        args = (_lib.ptr(target_logits), _lib.ptr(draft_logits), b, r, v, float(temperature), float(top_p),
                _lib.ptr(parent), _lib.ptr(n_rows), _lib.ptr(tokens), _lib.ptr(uniforms), uniforms.shape[1],
                _lib.ptr(self._ws), self._ws.numel(), _lib.ptr(o["path"]), _lib.ptr(o["path_len"]),
                _lib.ptr(o["next_token"]), _lib.ptr(o["used"]), _lib.ptr(o["residual"]), _lib.ptr(o["err"]),
                _lib.ptr(allowed), n_words)
        if lazy and levels:
            main = stream if stream is not None else torch.cuda.current_stream()
            if self._side is None or self._side.device != main.device:
                self._side = torch.cuda.Stream(device=main.device)
            self._side.wait_stream(main)  # err zeroed, inputs ready
            # every row checked beside the lazy walk (HBM-bound vs latency-bound)
            if not _DIAG_SKIP_VALIDATE:
                rc = lib.sdb_stochastic_validate(_lib.ptr(target_logits), _lib.ptr(draft_logits), b, r, v,
                                                 _lib.ptr(parent), _lib.ptr(n_rows), _lib.ptr(allowed), n_words,
                                                 _lib.ptr(o["err"]), _lib.stream_ptr(self._side))
                _lib.check(rc, "stochastic_validate")
            rc = lib.sdb_accept_stochastic_lazy(*args, int(levels), _lib.stream_ptr(main))
            _lib.check(rc, "accept_stochastic_lazy")
            main.wait_stream(self._side)
        else:
            rc = lib.sdb_accept_stochastic_ex(*args, _lib.stream_ptr(stream))
            _lib.check(rc, "accept_stochastic")
        return AcceptResult(o["path"], o["path_len"], o["next_token"], o["used"], o["err"], o["residual"])


def accept_stochastic(target_logits, draft_logits, temperature, top_p, parent, n_rows, tokens, uniforms=None,
                      want_residual=False, stream=None, seeds=None, steps=None, allowed=None):
    """Batched T > 0 acceptance (target_dist for every row, draft q per parent
    row, MSS walk).  uniforms float64 [B, n_uniforms] (the reference's
    rank_sliced_uniforms row per sequence), or ``uniforms=None`` with int64
    ``seeds``/``steps`` [B] to draw row 0 of the reference's Philox matrix on
    the device (engine.py:251-254)."""
    return StochasticAcceptor()(target_logits, draft_logits, temperature, top_p, parent, n_rows, tokens, uniforms,
                                want_residual, stream, seeds, steps, allowed)
