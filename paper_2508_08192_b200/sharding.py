"""Multi-GPU partitioning of the verify path (one process per GPU).

* Attention shards by KV head with no communication: rank r of G owns KV
  heads [r*Hkv/G, (r+1)*Hkv/G) and their q heads (GQA groups stay whole), for
  every page of every sequence (same block table on all ranks).
* Greedy acceptance shards the vocabulary (a column-parallel LM head leaves
  logits vocab-sharded): each rank packs (orderable max logit, ~global index)
  into one int64 per row (sdb_argmax_keys) and ONE all-reduce(MAX) over B*R
  keys yields the global argmax with the reference's lowest-index tie
  break (numcore.py:53); every rank then runs the same walk, so path / next
  token / compaction are replicated without a broadcast.

* Stochastic acceptance shards the vocabulary too (ShardedStochasticAcceptor):
  a fixed sequence of phase kernels (csrc/accept_sharded.cu) separated by
  small batched collectives (one all-gather, all-reduces SUM/MAX) -- global
  softmax statistics, the exact top-p cut by four byte-wise mass-histogram
  passes, the drafted tokens' p/q, the rejection chains of every parent row,
  then an identical walk on every rank and an owner-draws bonus token.

The reference has no distributed backend (it only simulates TP ranks for the
uniform stream, sampling.py:112-124); this is the B200 design of SURVEY.md
section 8(e).
"""

from __future__ import annotations

from dataclasses import dataclass


@dataclass(frozen=True)
class Shard:
    rank: int
    world: int
    kv_lo: int
    kv_hi: int
    q_lo: int
    q_hi: int
    v_lo: int
    v_hi: int
    vocab: int = 0  # global vocabulary size

    @property
    def n_kv(self):
        return self.kv_hi - self.kv_lo

    @property
    def n_q(self):
        return self.q_hi - self.q_lo

    @property
    def n_vocab(self):
        return self.v_hi - self.v_lo


def shard_for(rank, world, n_heads, n_kv_heads, vocab):
    """KV-head and vocabulary ranges owned by `rank` of `world`."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError("bad rank/world")
    if n_kv_heads % world:
        raise ValueError(f"{n_kv_heads} KV heads do not split over {world} ranks")
    if n_heads % n_kv_heads:
        raise ValueError("q heads must be a multiple of KV heads")
    g = n_heads // n_kv_heads
    per = n_kv_heads // world
    kv_lo = rank * per
    base, extra = divmod(vocab, world)
    v_lo = rank * base + min(rank, extra)
    v_hi = v_lo + base + (1 if rank < extra else 0)
    return Shard(rank, world, kv_lo, kv_lo + per, kv_lo * g, (kv_lo + per) * g, v_lo, v_hi, vocab)


def combine_argmax_keys(keys, group=None):
    """In-place all-reduce(MAX) of packed int64 argmax keys across ranks."""
    import torch.distributed as dist

    if dist.is_available() and dist.is_initialized() and dist.get_world_size(group) > 1:
        dist.all_reduce(keys, op=dist.ReduceOp.MAX, group=group)
    return keys


def key_to_index(keys):
    """Global token index from packed keys (low word = 0xFFFFFFFF - index)."""
    return 0xFFFFFFFF - (keys & 0xFFFFFFFF)


class ShardedGreedyAcceptor:
    """Vocab-sharded T = 0 acceptance: local keys -> all-reduce MAX -> walk."""

    def __init__(self, shard: Shard, group=None):
        self.shard = shard
        self.group = group

    def __call__(self, logits_shard, parent, n_rows, tokens, stream=None):
        """The rank's error word rides in the same all-reduce as the keys (one
        extra int64 after the B*R keys), so a NaN in any shard raises on every
        rank (softmax_lse, numcore.py:47-48) instead of only on its owner."""
        import torch

        from . import _lib
        from .sampling import greedy_walk

        b, r, v = logits_shard.shape
        if logits_shard.stride(2) != 1 or (b > 1 and logits_shard.stride(0) != r * logits_shard.stride(1)):
            raise ValueError("logits shard must be [B, R, V_local] with unit vocab stride and uniform row stride")
        rows = b * r
        dev = logits_shard.device
        keys = torch.empty((rows + 1,), dtype=torch.int64, device=dev)
        err = torch.zeros((1,), dtype=torch.int32, device=dev)
        dt = _lib.DTYPE_F32 if logits_shard.dtype == torch.float32 else _lib.DTYPE_BF16
        rc = _lib.lib().sdb_argmax_keys(_lib.ptr(logits_shard), dt, rows, v, logits_shard.stride(1),
                                        int(self.shard.v_lo), _lib.ptr(keys), _lib.ptr(err), _lib.stream_ptr(stream))
        _lib.check(rc, "argmax_keys")
        with torch.cuda.stream(stream if stream is not None else torch.cuda.current_stream(dev)):
            keys[rows:].copy_(err)  # error bits (MAX over ranks: nonzero anywhere -> nonzero everywhere)
            combine_argmax_keys(keys, self.group)
            res = greedy_walk(keys[:rows].reshape(b, r), parent, n_rows, tokens, stream=stream)
            res.err = keys[rows:].to(torch.int32)
        return res


class TorchComm:
    """Collectives of one rank over torch.distributed (NCCL in production,
    gloo in the CPU-side tests); operates on single-element tensor lists."""

    def __init__(self, group=None):
        import torch.distributed as dist

        self.dist = dist
        self.group = group
        self.world = dist.get_world_size(group) if dist.is_initialized() else 1
        self.rank = dist.get_rank(group) if dist.is_initialized() else 0

    def all_gather(self, outs, ins):
        (out,), (inp,) = outs, ins
        if self.world == 1:
            out[0].copy_(inp)
            return
        try:
            self.dist.all_gather_into_tensor(out, inp, group=self.group)
        except (RuntimeError, AttributeError, ValueError):
            self.dist.all_gather(list(out.unbind(0)), inp, group=self.group)

    def all_reduce_sum(self, ts):
        if self.world > 1:
            self.dist.all_reduce(ts[0], op=self.dist.ReduceOp.SUM, group=self.group)

    def all_reduce_max(self, ts):
        if self.world > 1:
            self.dist.all_reduce(ts[0], op=self.dist.ReduceOp.MAX, group=self.group)


class VirtualComm:
    """All `world` shards in one process (one GPU): the collectives are
    element-wise sums / maxima over the per-shard tensors.  Used by the GPU
    parity tests to run the exact multi-rank protocol on one device."""

    def all_gather(self, outs, ins):
        import torch

        st = torch.stack(list(ins), 0)
        for o in outs:
            o.copy_(st)

    def all_reduce_sum(self, ts):
        tot = ts[0].clone()
        for t in ts[1:]:
            tot += t
        for t in ts:
            t.copy_(tot)

    def all_reduce_max(self, ts):
        m = ts[0].clone()
        for t in ts[1:]:
            m = m.maximum(t)
        for t in ts:
            t.copy_(m)


def max_children(parent):
    """Largest number of children of any row (host sync; pass it explicitly
    when capturing a CUDA graph)."""
    import torch

    par = parent.long()
    b, r = par.shape
    valid = par >= 0
    flat = (par.clamp(min=0) + torch.arange(b, device=par.device)[:, None] * r)[valid]
    cnt = torch.bincount(flat, minlength=b * r)
    return int(cnt.max().item()) if cnt.numel() else 0


class _ShardCtx:
    """Exchange buffers + argument block of one rank's shard."""

    def __init__(self, shard: Shard, b, r, vl, vocab, levels, dev, want_residual):
        import torch

        from . import _lib

        self.shard = shard
        a = _lib.ShardedAcceptArgs()
        a.batch, a.r_max, a.vocab_local = b, r, vl
        a.vocab_offset, a.vocab = shard.v_lo, vocab
        a.world, a.rank = shard.world, shard.rank
        a.max_children = levels
        sizes = (_lib.I64 * _lib.SH_N_BUFS)()
        _lib.check(_lib.lib().sdb_sharded_accept_sizes(a, sizes), "sharded_accept_sizes")
        f64, i32, i64 = torch.float64, torch.int32, torch.int64
        self.partials = torch.zeros(sizes[0], dtype=f64, device=dev)
        self.gathered = torch.zeros((shard.world, sizes[0]), dtype=f64, device=dev)
        self.hist = torch.zeros(sizes[2], dtype=f64, device=dev)
        self.tie = torch.zeros(sizes[3], dtype=i32, device=dev)
        self.pq = torch.zeros(sizes[4], dtype=f64, device=dev)
        self.chain_x = torch.zeros(sizes[5], dtype=f64, device=dev)
        self.bonus_mass = torch.zeros(sizes[6], dtype=f64, device=dev)
        self.bonus_token = torch.zeros(sizes[7], dtype=i64, device=dev)
        self.scratch = torch.empty(sizes[8], dtype=torch.uint8, device=dev)
        self.path = torch.zeros((b, r), dtype=i32, device=dev)
        self.path_len = torch.zeros((b,), dtype=i32, device=dev)
        self.used = torch.zeros((b,), dtype=i32, device=dev)
        self.err = torch.zeros((1,), dtype=i32, device=dev)
        self.uni = torch.empty((b, r), dtype=f64, device=dev)
        self.residual = torch.empty((b, vl), dtype=torch.float32, device=dev) if want_residual else None
        a.xchg_partials, a.gathered, a.hist = (self.partials.data_ptr(), self.gathered.data_ptr(),
                                               self.hist.data_ptr())
        a.tie, a.pq, a.chain_x = self.tie.data_ptr(), self.pq.data_ptr(), self.chain_x.data_ptr()
        a.bonus_mass, a.bonus_token = self.bonus_mass.data_ptr(), self.bonus_token.data_ptr()
        a.scratch, a.scratch_bytes = self.scratch.data_ptr(), self.scratch.numel()
        a.path, a.path_len, a.uniforms_used = self.path.data_ptr(), self.path_len.data_ptr(), self.used.data_ptr()
        a.residual = self.residual.data_ptr() if self.residual is not None else None
        a.err = self.err.data_ptr()
        self.args = a

    def bind(self, target, draft, temperature, top_p, parent, n_rows, tokens, uniforms):
        a = self.args
        a.target_logits, a.draft_logits = target.data_ptr(), draft.data_ptr()
        a.temperature, a.top_p = float(temperature), float(top_p)
        a.parent, a.n_rows, a.tokens = parent.data_ptr(), n_rows.data_ptr(), tokens.data_ptr()
        a.uniforms, a.n_uniforms = uniforms.data_ptr(), uniforms.shape[1]


def run_sharded_stochastic(ctxs, comm, top_p, levels, stream=None):
    """The phase / collective sequence of csrc/accept_sharded.cu over the
    shard contexts `ctxs` (one per rank in this process)."""
    from . import _lib

    lib = _lib.lib()
    sp = _lib.stream_ptr(stream)

    def phase(ph, level=0):
        for c in ctxs:
            _lib.check(lib.sdb_sharded_accept_phase(c.args, ph, level, sp), f"sharded_accept phase {ph}")

    for c in ctxs:
        _lib.clear(c.err, stream)
    phase(_lib.SH_PARTIALS)
    comm.all_gather([c.gathered for c in ctxs], [c.partials for c in ctxs])
    phase(_lib.SH_COMBINE)
    if top_p < 1.0:
        for k in range(4):
            phase(_lib.SH_NUCLEUS, k)
            comm.all_reduce_sum([c.hist for c in ctxs])
        phase(_lib.SH_CUT)
        comm.all_reduce_sum([c.tie for c in ctxs])
        phase(_lib.SH_FINISH)
    phase(_lib.SH_TOKEN_PQ)
    comm.all_reduce_sum([c.pq for c in ctxs])
    for k in range(1, levels + 1):
        phase(_lib.SH_RESIDUAL, k)
        comm.all_reduce_sum([c.chain_x for c in ctxs])
    phase(_lib.SH_WALK)
    comm.all_reduce_sum([c.bonus_mass for c in ctxs])
    phase(_lib.SH_PICK)
    comm.all_reduce_max([c.bonus_token for c in ctxs])


class ShardedStochasticAcceptor:
    """Vocab-sharded T > 0 acceptance of this rank's logits slice: same call
    signature and results as sampling.StochasticAcceptor (path, path_len,
    next_token, uniforms_used identical on every rank)."""

    def __init__(self, shard: Shard, group=None, max_children=None):
        self.shard = shard
        self.comm = TorchComm(group)
        self.levels = max_children
        self._ctx = None

    def __call__(self, target_logits, draft_logits, temperature, top_p, parent, n_rows, tokens, uniforms=None,
                 want_residual=False, stream=None, seeds=None, steps=None):
        import torch

        from .sampling import AcceptResult, SamplingError, device_uniforms

        b, r, vl = target_logits.shape
        if vl != self.shard.n_vocab:
            raise SamplingError(f"logits slice has {vl} columns, shard owns {self.shard.n_vocab}")
        if target_logits.dtype != torch.float32 or draft_logits.dtype != torch.float32:
            raise SamplingError("stochastic acceptance takes fp32 logits")
        if not target_logits.is_contiguous() or not draft_logits.is_contiguous():
            raise SamplingError("logits slices must be contiguous [B, R, V_local]")
        if not (temperature > 0):
            raise SamplingError("stochastic acceptance needs temperature > 0 (use accept_greedy)")
        levels = self.levels if self.levels is not None else max_children(parent)
        key = (b, r, vl, levels, str(target_logits.device), want_residual)
        if self._ctx is None or self._ctx[0] != key:
            self._ctx = (key, _ShardCtx(self.shard, b, r, vl, self.shard.vocab, levels, target_logits.device,
                                        want_residual))
        ctx = self._ctx[1]
        if uniforms is None:
            if seeds is None or steps is None:
                raise SamplingError("pass uniforms, or seeds and steps")
            uniforms = device_uniforms(seeds, steps, r, out=ctx.uni, stream=stream)
        ctx.bind(target_logits, draft_logits, temperature, top_p, parent, n_rows, tokens, uniforms)
        run_sharded_stochastic([ctx], self.comm, float(top_p), levels, stream)
        return AcceptResult(ctx.path, ctx.path_len, ctx.bonus_token, ctx.used, ctx.err, ctx.residual)


def run_virtual_sharded_stochastic(target_logits, draft_logits, temperature, top_p, parent, n_rows, tokens, uniforms,
                                   world, want_residual=False, max_children_=None):
    """Test/diagnostic driver: split full-vocab logits into `world` shards and
    run every rank's kernels in this process with VirtualComm.  Returns the
    per-rank results."""
    from .sampling import AcceptResult

    b, r, vocab = target_logits.shape
    levels = max_children_ if max_children_ is not None else max_children(parent)
    ctxs, slices = [], []
    for rank in range(world):
        sh = shard_for(rank, world, world, world, vocab)
        t = target_logits[:, :, sh.v_lo:sh.v_hi].contiguous()
        d = draft_logits[:, :, sh.v_lo:sh.v_hi].contiguous()
        c = _ShardCtx(sh, b, r, sh.n_vocab, vocab, levels, target_logits.device, want_residual)
        c.bind(t, d, temperature, top_p, parent, n_rows, tokens, uniforms)
        ctxs.append(c)
        slices.append((t, d))
    run_sharded_stochastic(ctxs, VirtualComm(), float(top_p), levels)
    return [AcceptResult(c.path, c.path_len, c.bonus_token, c.used, c.err, c.residual) for c in ctxs]
