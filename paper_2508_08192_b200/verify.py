"""The batched tree-verification step on one GPU (or one KV-head shard).

One step = what Engine.validate_stage + the sample/bookkeep stages do per
round for the whole batch on one attention layer (engine.py:447-523):

  1. tree_build      -- ancestor mask words / positions from the parent arrays
  2. tree attention  -- prefix over the paged KV + masked suffix + LSE merge
  3. acceptance      -- greedy (T = 0) or stochastic (T > 0) over the logits
  4. compact_kv      -- accepted rows' K/V into the sequence's pages

All four are device launches on the caller's stream with no host sync, so
the step can be captured into a CUDA graph (``capture``).
"""

from __future__ import annotations

from dataclasses import dataclass

from . import _lib
from .attention import TreeVerifyAttention
from .drafttree import n_words
from .kvstore import compact_kv
from .sampling import GreedyAcceptor, StochasticAcceptor


@dataclass
class StepInputs:
    parent: "object"       # int32 [B, R] augmented parents
    n_rows: "object"       # int32 [B]
    ctx_len: "object"      # int32 [B] committed rows in cache (L - 1)
    tokens: "object"       # int32 [B, R] row tokens (row 0 = root)
    q: "object"            # [B, R, Hq, d]
    tree_k: "object"       # [B, R, Hkv, d]
    tree_v: "object"
    logits: "object"       # [B, R, V] target logits (vocab shard)
    k_pool: "object"       # [num_blocks, Hkv, bs, d] (one layer)
    v_pool: "object"
    block_table: "object"  # int32 [B, max_blocks]
    draft_logits: "object" = None  # [B, R, V] for stochastic acceptance
    uniforms: "object" = None      # float64 [B, n_uniforms]
    seeds: "object" = None         # int64 [B] Philox keys (uniforms=None: drawn on the device)
    steps: "object" = None         # int64 [B]
    allowed: "object" = None       # int32 [B, R, ceil(V/32)] FSM allowed-token words (sampling.pack_allowed)


_SMS = {}


def _num_sms(device):
    import torch

    if device not in _SMS:
        _SMS[device] = torch.cuda.get_device_properties(device).multi_processor_count
    return _SMS[device]


class TreeVerifier:
    def __init__(self, scale, temperature=0.0, top_p=1.0, max_ctx=None, num_splits=0, kernel=0, fuse_greedy=True,
                 chunk_len=None, reserve_sms=None, tree_levels=None):
        self.scale = scale
        self.temperature = temperature
        self.top_p = top_p
        self.max_ctx = max_ctx
        self.num_splits = num_splits
        self.kernel = kernel
        self.chunk_len = chunk_len  # iRoPE local chunk (tree truncated at the boundary by the caller)
        self.reserve_sms = reserve_sms  # SMs kept free of the attention for the concurrent acceptance (None: auto)
        self.fuse_greedy = fuse_greedy  # greedy scan inside the attention kernel: True (when it hides), "always", False
        self.attn = TreeVerifyAttention()
        self.greedy = GreedyAcceptor()
        # lazy stochastic acceptance needs the tree depth + 1 to be capturable
        self.stochastic = StochasticAcceptor(levels=tree_levels)
        self._out = None
        self._side = None
        self.graph = None

    def _buffers(self, x: StepInputs):
        import torch

        b, r, hq, d = x.q.shape
        key = (b, r, hq, d, x.q.dtype, str(x.q.device))
        if self._out is None or self._out[0] != key:
            dev = x.q.device
            w = n_words(r)
            self._out = (key, dict(
                mask=torch.empty((b, r, w), dtype=torch.int32, device=dev),
                pos=torch.empty((b, r), dtype=torch.int32, device=dev),
                depth=torch.empty((b, r), dtype=torch.int32, device=dev),
                tree_err=torch.empty((b,), dtype=torch.int32, device=dev),
                # sticky (no per-step clear launch): set by the attention when a
                # ctx_len exceeds max_ctx, reset by check()
                attn_err=torch.zeros((1,), dtype=torch.int32, device=dev),
                out=torch.empty_like(x.q),
                lse=torch.empty((b, hq, r), dtype=torch.float32, device=dev)))
        return self._out[1]

    def step(self, x: StepInputs, stream=None, compact=True, overlap=True):
        """One verification step.  Attention (tree_build -> attention) and
        acceptance (-> compaction) do not depend on each other, so with
        ``overlap`` they run as two branches (side stream forked from and
        joined back into ``stream``; captured as parallel graph branches):
        at small batches the attention leaves SMs idle that the acceptance
        kernels use."""
        import torch

        o = self._buffers(x)
        b, r = x.parent.shape
        lib = _lib.lib()
        main = stream if stream is not None else torch.cuda.current_stream()
        attn_args = (x.q, x.k_pool, x.v_pool, x.block_table, x.ctx_len, x.tree_k, x.tree_v, o["mask"], x.n_rows,
                     self.scale)
        attn_kw = dict(out=o["out"], lse=o["lse"], max_ctx=self.max_ctx, num_splits=self.num_splits,
                       kernel=self.kernel, chunk_len=self.chunk_len, err=o["attn_err"])
        # small batches: the attention's persistent grid leaves SMs free ->
        # run acceptance beside it; full occupancy -> fold the greedy scan
        # into the attention kernel (its otherwise idle warp + TMA ring)
        n_sms = _num_sms(main.device)
        attn_sms = self.attn.sms(*attn_args, **attn_kw)
        reserve = self.reserve_sms
        if reserve is None:
            reserve = self._auto_reserve(x, b, r, n_sms)
        if (overlap and reserve and attn_sms + 16 > n_sms and self.num_splits == 0
                and not (self.fuse_greedy and self.temperature == 0 and x.allowed is None
                         and self._scan_hides(x, b, r, main.device))):
            # full occupancy: shrink the attention's persistent grid so the
            # HBM-bound acceptance streams beside the tensor-bound attention
            group = max(1, self.attn.sms(*attn_args, **dict(attn_kw, num_splits=1)))  # SMs per worker
            # an even worker count keeps the two row blocks of a KV head in
            # step (an odd count misaligns them: K/V read twice; C3 with 63
            # pairs measured 693 us vs 646-657 with 62 / 64)
            attn_kw["num_splits"] = max(2, ((n_sms - reserve) // group) & ~1)
            attn_sms = self.attn.sms(*attn_args, **attn_kw)
        can_overlap = overlap and attn_sms + 16 <= n_sms
        fused = None
        if (not can_overlap and self.fuse_greedy and self.temperature == 0 and isinstance(self.greedy, GreedyAcceptor)
                and x.allowed is None
                and x.logits.dtype == torch.float32 and x.logits.stride(2) == 1
                and (self.fuse_greedy == "always" or self._scan_hides(x, b, r, main.device))):
            keys, err = self.greedy.fused_keys(b, r, x.logits.device)
            _lib.clear(err, main)  # before tree_build: the attention is tree_build's programmatic dependent
            fused = (x.logits, keys, err, 0)
        fork = torch.cuda.Event()
        fork.record(main)
        rc = lib.sdb_tree_build(_lib.ptr(x.parent), _lib.ptr(x.n_rows), _lib.ptr(x.ctx_len), b, r,
                                o["mask"].shape[-1], _lib.ptr(o["mask"]), _lib.ptr(o["pos"]), _lib.ptr(o["depth"]),
                                _lib.ptr(o["tree_err"]), _lib.stream_ptr(main))
        _lib.check(rc, "tree_build")
        self.attn(*attn_args, **attn_kw, stream=main, after_tree_build=True, fused_argmax=fused)
        if fused is not None:
            # the attention kernel streamed the logits and left the argmax keys
            acc = self.greedy.walk(x.parent, x.n_rows, x.tokens, stream=main)
            if compact:
                compact_kv(x.tree_k.unsqueeze(0), x.tree_v.unsqueeze(0), x.k_pool.unsqueeze(0),
                           x.v_pool.unsqueeze(0), x.block_table, x.ctx_len, acc.path, acc.path_len, None,
                           stream=main, err=acc.err)
            return o["out"], o["lse"], acc, o["tree_err"]
        # overlap only when the attention's persistent grid leaves SMs free
        # (small batches); at full occupancy the acceptance CTAs would delay
        # the attention's workers instead
        side = main
        if can_overlap:
            if self._side is None or self._side.device != main.device:
                self._side = torch.cuda.Stream(device=main.device)
            side = self._side
            side.wait_event(fork)
        with torch.cuda.stream(side):
            if self.temperature == 0:
                acc = (self.greedy(x.logits, x.parent, x.n_rows, x.tokens, stream=side) if x.allowed is None else
                       self.greedy(x.logits, x.parent, x.n_rows, x.tokens, stream=side, allowed=x.allowed))
            else:
                acc = self.stochastic(x.logits, x.draft_logits, self.temperature, self.top_p, x.parent, x.n_rows,
                                      x.tokens, x.uniforms, stream=side, seeds=x.seeds, steps=x.steps,
                                      **({} if x.allowed is None else {"allowed": x.allowed}))
            if compact:
                # writes cache rows >= ctx_len only: disjoint from what the
                # attention reads (prefix keys < ctx_len are the only unmasked ones)
                compact_kv(x.tree_k.unsqueeze(0), x.tree_v.unsqueeze(0), x.k_pool.unsqueeze(0),
                           x.v_pool.unsqueeze(0), x.block_table, x.ctx_len, acc.path, acc.path_len, None,
                           stream=side, err=acc.err)
        if side is not main:
            main.wait_stream(side)
        return o["out"], o["lse"], acc, o["tree_err"]

    def check(self, tree_err=None, acc=None):
        """Host sync: raise the reference exceptions for the last step's
        device error words -- TreeError (bad parent), CacheError (a ctx_len
        past ``max_ctx``: the attention plan would have dropped keys), and
        the acceptance's errors when ``acc`` is given."""
        from .drafttree import TreeError
        from .kvstore import CacheError

        o = self._out[1] if self._out is not None else None
        if o is None:
            return
        te = o["tree_err"] if tree_err is None else tree_err
        if int((te & _lib.SDB_ERR_BAD_PARENT).sum().item()):
            raise TreeError("parent must precede node or be ROOT")
        if int(o["attn_err"][0].item()) & _lib.SDB_ERR_CACHE:
            o["attn_err"].zero_()
            raise CacheError(f"context longer than max_ctx={self.max_ctx}: size TreeVerifier(max_ctx=) for the "
                             "longest sequence")
        if acc is not None:
            acc.raise_if_error()

    def _auto_reserve(self, x, b, r, n_sms):
        """SMs to leave to a greedy acceptance running beside a full-occupancy
        attention: k such that the scan on k SMs (~80 GB/s each, measured)
        takes as long as the attention on n_sms - k (~1.1 PFLOP/s on all
        SMs, measured).  C3: k = 20 (64 CTA pairs; step 690 -> ~640 us).  Stochastic
        acceptance is instruction-bound on every SM: no reserve."""
        import torch

        if self.temperature != 0 or x.logits.dtype != torch.float32:
            return 0
        hq, d = x.q.shape[2], x.q.shape[3]
        ctx = self.max_ctx if self.max_ctx else x.block_table.shape[1] * x.k_pool.shape[2]
        t_att = 4.0 * d * hq * b * r * ctx / 1.1e15
        # scan time on one SM: 90 GB/s per SM (the C3 step measures best at
        # 64 pairs / 20 SMs left, 629-649 us, vs 641-665 at 62 / 22 on the
        # same boxes; the 80 GB/s measured alone under-states the rate)
        acc_sm_s = b * r * x.logits.shape[2] * 4 / 90.0e9
        # acc_sm_s / k = t_att * n / (n - k)  ->  k = acc_sm_s * n / (t_att * n + acc_sm_s)
        k = acc_sm_s * n_sms / (t_att * n_sms + acc_sm_s)
        k = int(round(k))
        return k if 8 <= k <= n_sms // 2 else 0

    def _scan_hides(self, x, b, r, device):
        """Fold the greedy scan into the attention kernel only when one warp
        per CTA streaming its share of the logits (~10 GB/s per SM through
        the 40 KB TMA ring, measured) finishes well inside the attention
        (~1 PFLOP/s achieved): e.g. 405B shapes (C4) yes, 70B bs32 (C3) no."""
        hq, d = x.q.shape[2], x.q.shape[3]
        ctx = self.max_ctx if self.max_ctx else x.block_table.shape[1] * x.k_pool.shape[2]
        attn_s = 4.0 * d * hq * b * r * ctx / 1.0e15
        scan_s = (b * r / _num_sms(device)) * x.logits.shape[2] * 4 / 10.0e9
        return scan_s < 0.8 * attn_s

    def capture(self, x: StepInputs, warmup=2):
        """Capture one step into a CUDA graph; replay with ``replay()``."""
        import torch

        s = torch.cuda.Stream()
        s.wait_stream(torch.cuda.current_stream())
        with torch.cuda.stream(s):
            for _ in range(warmup):
                self.step(x, stream=s)
        torch.cuda.current_stream().wait_stream(s)
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g):
            res = self.step(x, stream=torch.cuda.current_stream())
        self.graph = g
        self.graph_outputs = res
        return res

    def replay(self):
        self.graph.replay()
        return self.graph_outputs


_BATCH_FIELDS = ("parent", "n_rows", "ctx_len", "tokens", "q", "tree_k", "tree_v", "logits", "block_table",
                 "draft_logits", "uniforms", "seeds", "steps", "allowed")


def _slice_inputs(x: StepInputs, b0: int, b1: int) -> StepInputs:
    """The sequences [b0, b1) of a step (batch-major views; the KV pools are shared)."""
    f = {k: getattr(x, k) for k in StepInputs.__dataclass_fields__}
    for k in _BATCH_FIELDS:
        if f[k] is not None:
            f[k] = f[k][b0:b1]
    return StepInputs(**f)


class HostStepPipeline:
    """One verification step from pinned HOST inputs to pinned HOST outputs
    (the reference engine's data lives on the host), pipelined over chunks of
    sequences: chunk c's host->device copies (a copy stream) overlap chunk
    c - 1's step (the compute stream) and chunk c - 2's device->host copies
    (a third stream; PCIe is full duplex), so a step costs the H2D of its
    inputs plus the step and D2H of the LAST chunk only.  Each chunk has its
    own TreeVerifier (own output buffers: chunk c + 1's step must not
    overwrite what chunk c's D2H is still reading).

    ``x_dev``: the device StepInputs (resident KV pools + per-step buffers
    that the copies land in); ``host_in``: field name -> pinned host tensor
    (batch-major, same shape as the device field); ``host_out``: any of
    "out", "lse", "path", "path_len", "next_token" -> pinned host tensor."""

    def __init__(self, make_verifier, chunks=4):
        self.make_verifier = make_verifier
        self.chunks = max(1, int(chunks))
        self.verifiers = None
        self._streams = None

    def __call__(self, x_dev: StepInputs, host_in: dict, host_out: dict, stream=None):
        import torch

        main = stream if stream is not None else torch.cuda.current_stream()
        b = x_dev.parent.shape[0]
        n = min(self.chunks, b)
        if self.verifiers is None or len(self.verifiers) != n:
            self.verifiers = [self.make_verifier() for _ in range(n)]
            self.accs = [None] * n
        if self._streams is None or self._streams[0].device != main.device:
            self._streams = (torch.cuda.Stream(device=main.device), torch.cuda.Stream(device=main.device))
        h2d, d2h = self._streams
        bounds = [(b * c // n, b * (c + 1) // n) for c in range(n)]
        h2d.wait_stream(main)  # the previous step's users of the input buffers are done
        d2h.wait_stream(main)
        last = None
        for c, (b0, b1) in enumerate(bounds):
            with torch.cuda.stream(h2d):
                for k, v in host_in.items():
                    getattr(x_dev, k)[b0:b1].copy_(v[b0:b1], non_blocking=True)
                landed = torch.cuda.Event()
                landed.record(h2d)
            main.wait_event(landed)
            out, lse, acc, _ = self.verifiers[c].step(_slice_inputs(x_dev, b0, b1), stream=main)
            done = torch.cuda.Event()
            done.record(main)
            d2h.wait_event(done)
            res = {"out": out, "lse": lse, "path": acc.path, "path_len": acc.path_len, "next_token": acc.next_token}
            with torch.cuda.stream(d2h):
                for k, t in host_out.items():
                    t[b0:b1].copy_(res[k], non_blocking=True)
            last = (out, lse, acc)
            self.accs[c] = acc
        main.wait_stream(d2h)
        main.wait_stream(h2d)
        return last

    def check(self):
        """Raise the reference exceptions for every chunk's device error words."""
        for v, a in zip(self.verifiers or (), self.accs or ()):
            v.check(acc=a)
