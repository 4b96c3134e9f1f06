"""Tree attention: the reference's op API on the GPU, plus the batched
paged GQA tree-verify operator.

Drop-in layer (numpy float64 in/out, reference semantics and errors):
``attend``, ``merge_partials``, ``merge_attentions``, ``tree_attention``,
``explicit_tree_mask``, ``naive_tree_attention``,
``truncate_draft_at_boundary`` -- attention.py:20-206 of the reference.  The
arithmetic runs in float64 on the device (sdb_attend_heads_f64,
sdb_merge_partials_f64) so the reference's own tolerances (1e-12 / 1e-10)
hold.  GQA is an extra keyword ``n_kv_heads`` (defaults to ``n_heads``).

Perf layer: ``tree_verify_attention`` -- one launch computes, for every
sequence of the batch and every q head, prefix attention over the paged KV
cache + masked suffix attention over the fresh tree K/V + their LSE merge
(model.py:252-272) in bf16 with fp32 accumulation.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from . import _lib
from .drafttree import TreeSpec, suffix_mask


class AttentionError(ValueError):
    pass


@dataclass(frozen=True)
class CausalPrefix:
    context_len: int


@dataclass(frozen=True)
class LocalChunk:
    chunk_len: int
    q_positions: tuple
    k_positions: tuple


@dataclass(frozen=True)
class TreeSuffix:
    mask: np.ndarray


@dataclass
class PartialAttention:
    out: np.ndarray  # (queries, dim)
    lse: np.ndarray  # (heads, queries); -inf marks fully-masked rows

    @property
    def masked_rows(self):
        return ~np.isfinite(self.lse)


def _as_matrix(x):
    a = np.asarray(x, dtype=np.float64)
    if a.ndim != 2:
        raise ValueError(f"expected 2-D matrix, got shape {a.shape}")
    return a


def _split_heads(x, n_heads):
    rows, dim = x.shape
    if dim % n_heads != 0:
        raise AttentionError(f"dim {dim} not divisible by {n_heads} heads")
    return np.ascontiguousarray(x.reshape(rows, n_heads, dim // n_heads).transpose(1, 0, 2))


def _join_heads(x):
    heads, rows, dh = x.shape
    return np.ascontiguousarray(x.transpose(1, 0, 2)).reshape(rows, heads * dh)


def _bias_kind(bias):
    """Bias class by name, so the reference's own CausalPrefix / LocalChunk /
    TreeSuffix objects (attention.py:24-47) work when this module replaces
    the reference's ``attend`` in place (shim.install_reference)."""
    kind = type(bias).__name__
    return kind if kind in ("CausalPrefix", "LocalChunk", "TreeSuffix") else None


def _bias_mask(bias, n_q, n_k):
    """Visibility matrix for a bias object (attention.py:76-90)."""
    kind = _bias_kind(bias)
    if kind == "CausalPrefix":
        if bias.context_len != n_k:
            raise AttentionError("CausalPrefix context_len must match key count")
        return None
    if kind == "LocalChunk":
        if bias.chunk_len < 1:
            raise AttentionError("LocalChunk chunk_len must be >= 1")
        qp = np.asarray(bias.q_positions)
        kp = np.asarray(bias.k_positions)
        if qp.shape != (n_q,) or kp.shape != (n_k,):
            raise AttentionError("LocalChunk positions must match q/k lengths")
        same = qp[:, None] // bias.chunk_len == kp[None, :] // bias.chunk_len
        return same & (kp[None, :] <= qp[:, None])
    if kind == "TreeSuffix":
        if bias.mask.shape != (n_q, n_k):
            raise AttentionError(f"TreeSuffix mask {bias.mask.shape} vs ({n_q}, {n_k})")
        return np.asarray(bias.mask, dtype=bool)
    raise AttentionError(f"unknown bias {bias!r}")


def attend_heads(q, k, v, mask, scale):
    """Device float64 attention core: q (H, m, d), k/v (H, n, d), mask (m, n)
    bool or None -> (out (H, m, d), lse (H, m)).  Replaces
    kernels.attend_heads (kernels.py:195-203)."""
    import torch

    q = np.ascontiguousarray(q, dtype=np.float64)
    k = np.ascontiguousarray(k, dtype=np.float64)
    v = np.ascontiguousarray(v, dtype=np.float64)
    h, m, d = q.shape
    n = k.shape[1]
    dev = "cuda"
    tq, tk, tv = (torch.from_numpy(x).to(dev) for x in (q, k, v))
    tm = None if mask is None else torch.from_numpy(np.ascontiguousarray(mask, dtype=np.uint8)).to(dev)
    out = torch.empty((h, m, d), dtype=torch.float64, device=dev)
    lse = torch.empty((h, m), dtype=torch.float64, device=dev)
    rc = _lib.lib().sdb_attend_heads_f64(_lib.ptr(tq), _lib.ptr(tk), _lib.ptr(tv), _lib.ptr(tm), h, m, n, d,
                                         float(scale), _lib.ptr(out), _lib.ptr(lse), _lib.stream_ptr())
    _lib.check(rc, "attend_heads")
    return out.cpu().numpy(), lse.cpu().numpy()


def _gqa_expand(x, n_heads, n_kv_heads):
    if n_kv_heads == n_heads:
        return x
    if n_heads % n_kv_heads:
        raise AttentionError(f"{n_heads} q heads not divisible by {n_kv_heads} kv heads")
    rows, dim = x.shape
    d = dim // n_kv_heads
    g = n_heads // n_kv_heads
    return np.repeat(x.reshape(rows, n_kv_heads, d), g, axis=1).reshape(rows, n_heads * d)


def attend(q, k, v, bias, scale, n_heads=1, n_kv_heads=None):
    """softmax(q k^T * scale + mask) v with per-query LSE (attention.py:92-105)."""
    q, k, v = _as_matrix(q), _as_matrix(k), _as_matrix(v)
    n_kv = n_heads if n_kv_heads is None else n_kv_heads
    if k.shape != v.shape or q.shape[1] // n_heads != k.shape[1] // max(n_kv, 1) or q.shape[1] % n_heads:
        raise AttentionError(f"attend: q {q.shape}, k {k.shape}, v {v.shape}")
    k, v = _gqa_expand(k, n_heads, n_kv), _gqa_expand(v, n_heads, n_kv)
    if q.shape[1] != k.shape[1]:
        raise AttentionError(f"attend: q {q.shape}, k {k.shape}, v {v.shape}")
    n_q, n_k = q.shape[0], k.shape[0]
    if n_k == 0:
        return PartialAttention(np.zeros((n_q, q.shape[1])), np.full((n_heads, n_q), -np.inf))
    mask = _bias_mask(bias, n_q, n_k)
    out, lse = attend_heads(_split_heads(q, n_heads), _split_heads(k, n_heads), _split_heads(v, n_heads), mask,
                            scale)
    return PartialAttention(_join_heads(out), lse)


def merge_partials(parts, n_heads=1):
    """LSE merge of disjoint-key partials on the device (attention.py:108-124)."""
    import torch

    if not parts:
        raise AttentionError("merge: no parts")
    lses = np.ascontiguousarray(np.stack([p.lse for p in parts]), dtype=np.float64)
    outs = np.ascontiguousarray(np.stack([_split_heads(_as_matrix(p.out), n_heads) for p in parts]))
    n_parts, h, m, d = outs.shape
    to = torch.from_numpy(outs).cuda()
    tl = torch.from_numpy(lses).cuda()
    out = torch.empty((h, m, d), dtype=torch.float64, device="cuda")
    lse = torch.empty((h, m), dtype=torch.float64, device="cuda")
    err = torch.zeros((1,), dtype=torch.int32, device="cuda")
    rc = _lib.lib().sdb_merge_partials_f64(_lib.ptr(to), _lib.ptr(tl), n_parts, h, m, d, _lib.ptr(out),
                                           _lib.ptr(lse), _lib.ptr(err), _lib.stream_ptr())
    _lib.check(rc, "merge_partials")
    if int(err.item()) & _lib.SDB_ERR_ALL_MASKED:
        raise AttentionError("merge: query row masked in every part")
    return PartialAttention(_join_heads(out.cpu().numpy()), lse.cpu().numpy())


def merge_attentions(parts, n_heads=1):
    return merge_partials(parts, n_heads).out


def tree_attention(q_tree, committed_k, committed_v, tree_k, tree_v, tree, scale, n_heads=1, chunk_len=None,
                   n_kv_heads=None):
    """Two-pass tree attention (attention.py:131-151), GQA-capable."""
    ctx = committed_k.shape[0]
    if q_tree.shape[0] != tree.n_nodes or tree_k.shape[0] != tree.n_nodes:
        raise AttentionError("tree_attention: node count mismatch")
    q_pos = tuple(ctx + d - 1 for d in tree.depth)
    prefix_bias = CausalPrefix(ctx) if chunk_len is None else LocalChunk(chunk_len, q_pos, tuple(range(ctx)))
    parts = []
    if ctx > 0:
        parts.append(attend(q_tree, committed_k, committed_v, prefix_bias, scale, n_heads, n_kv_heads))
    parts.append(attend(q_tree, tree_k, tree_v, TreeSuffix(suffix_mask(tree)), scale, n_heads, n_kv_heads))
    return merge_attentions(parts, n_heads)


def explicit_tree_mask(tree, context_len, chunk_len=None):
    """Full (nodes, context+nodes) visibility (attention.py:154-169)."""
    n = tree.n_nodes
    mask = np.zeros((n, context_len + n), dtype=bool)
    q_pos = np.array([context_len + d - 1 for d in tree.depth], dtype=np.int64)
    k_pos = np.arange(context_len, dtype=np.int64)
    if chunk_len is None:
        mask[:, :context_len] = True
    else:
        mask[:, :context_len] = q_pos[:, None] // chunk_len == k_pos[None, :] // chunk_len
    mask[:, context_len:] = suffix_mask(tree)
    return mask


def naive_tree_attention(q_tree, full_k, full_v, explicit_mask, scale, n_heads=1):
    """One-pass explicit-mask attention (attention.py:172-186)."""
    q_tree, full_k, full_v = _as_matrix(q_tree), _as_matrix(full_k), _as_matrix(full_v)
    if explicit_mask.shape != (q_tree.shape[0], full_k.shape[0]):
        raise AttentionError("naive_tree_attention: mask shape mismatch")
    out, lse = attend_heads(_split_heads(q_tree, n_heads), _split_heads(full_k, n_heads),
                            _split_heads(full_v, n_heads), explicit_mask, scale)
    if not np.isfinite(lse).all():
        raise AttentionError("naive_tree_attention: fully masked query row")
    return _join_heads(out)


def truncate_draft_at_boundary(tree, committed_len, chunk_len):
    """Drop nodes crossing the iRoPE chunk boundary (attention.py:189-206)."""
    if chunk_len is None:
        return tree
    if chunk_len < 1:
        raise AttentionError("chunk_len must be >= 1")
    boundary = ((committed_len - 1) // chunk_len + 1) * chunk_len
    keep = [i for i, d in enumerate(tree.depth) if committed_len + d - 1 < boundary]
    if len(keep) == tree.n_nodes:
        return tree
    from .drafttree import subtree

    return subtree(tree, keep)[0]


# ---------------------------------------------------------------------------
# batched device operator
# ---------------------------------------------------------------------------

KERNEL_AUTO, KERNEL_TCGEN05, KERNEL_SIMT = 0, 1, 2


class TreeVerifyAttention:
    """Reusable launcher for sdb_tree_attn with a cached workspace, so a step
    can be captured in a CUDA graph (no allocation inside the launch)."""

    def __init__(self):
        self._ws = None
        self.last_sms = None

    def _args(self, q, k_cache, v_cache, block_table, ctx_len, tree_k, tree_v, mask_words, n_rows, scale,
                 out=None, lse=None, max_ctx=None, num_splits=0, kernel=KERNEL_AUTO, stream=None, q_row0=None,
                 max_q_nodes=None, after_tree_build=False, fused_argmax=None, chunk_len=None, err=None):
        import torch

        b, r, hq, d = q.shape
        nb, hkv, bs, d2 = k_cache.shape
        if d2 != d or tree_k.shape != (b, r, hkv, d):
            raise AttentionError("tree_verify_attention: shape mismatch")
        if q.dtype == torch.bfloat16:
            dt = _lib.DTYPE_BF16
        elif q.dtype == torch.float32:
            dt = _lib.DTYPE_F32
        else:
            raise AttentionError(f"unsupported dtype {q.dtype}")
        for t in (k_cache, v_cache, tree_k, tree_v):
            if t.dtype != q.dtype or not t.is_contiguous():
                raise AttentionError("q/k/v must share dtype and be contiguous")
        if out is None:
            out = torch.empty_like(q)
        if lse is None:
            lse = torch.empty((b, hq, r), dtype=torch.float32, device=q.device)
        a = _lib.TreeAttnArgs()
        a.q, a.k_cache, a.v_cache = q.data_ptr(), k_cache.data_ptr(), v_cache.data_ptr()
        a.block_table, a.ctx_len = block_table.data_ptr(), ctx_len.data_ptr()
        a.tree_k, a.tree_v = tree_k.data_ptr(), tree_v.data_ptr()
        a.mask_words, a.n_rows = mask_words.data_ptr(), n_rows.data_ptr()
        a.out, a.lse = out.data_ptr(), lse.data_ptr()
        a.batch, a.r_max, a.n_words, a.hq, a.hkv, a.head_dim = b, r, mask_words.shape[-1], hq, hkv, d
        a.block_size, a.num_blocks, a.max_blocks = bs, nb, block_table.shape[1]
        a.max_ctx = int(max_ctx) if max_ctx is not None else block_table.shape[1] * bs
        a.scale, a.dtype, a.num_splits, a.kernel = float(scale), dt, int(num_splits), int(kernel)
        if q_row0 is not None:
            if q_row0.dtype != torch.int32 or q_row0.shape != (b,):
                raise AttentionError("q_row0 must be int32 [B]")
            a.q_row0 = q_row0.data_ptr()
        if max_q_nodes is not None:
            a.max_q_nodes = int(max_q_nodes)
        if chunk_len:  # iRoPE: every row sees prefix keys [floor(C / chunk) * chunk, C)
            a.chunk_len = int(chunk_len)
        if err is not None:  # int32 [1]: SDB_ERR_CACHE when a ctx_len exceeds max_ctx (keys would be dropped)
            if err.dtype != torch.int32 or err.numel() < 1:
                raise AttentionError("err must be an int32 tensor with >= 1 element")
            a.err = err.data_ptr()
        if after_tree_build:  # the previous kernel on `stream` is tree_build: PDL launch
            a.flags |= _lib.ATTN_FLAG_PDL
        if fused_argmax is not None:
            # (logits fp32 [B, R, V_local] (unit vocab stride), keys int64 [B*R], err int32 [1], vocab_offset)
            lg, keys, err, voff = fused_argmax
            if lg.dtype != torch.float32 or lg.stride(2) != 1 or lg.shape[:2] != (b, r):
                raise AttentionError("fused argmax: logits must be fp32 [B, R, V] with unit vocab stride")
            a.fused_logits, a.fused_row_stride, a.fused_vocab = lg.data_ptr(), lg.stride(1), lg.shape[2]
            a.fused_vocab_offset, a.fused_keys, a.fused_err = int(voff), keys.data_ptr(), err.data_ptr()
        return a, out, lse

    def sms(self, *args, **kw):
        """SMs the launch plan of this call would occupy (no launch)."""
        a, _, _ = self._args(*args, **kw)
        return _lib.lib().sdb_tree_attn_sms(a)

    def __call__(self, *args, **kw):
        import torch

        a, out, lse = self._args(*args, **kw)
        q = args[0]
        stream = kw.get("stream")
        lib = _lib.lib()
        self.last_sms = lib.sdb_tree_attn_sms(a)  # SMs this launch occupies (verify.TreeVerifier overlap)
        need = lib.sdb_tree_attn_workspace(a)
        if need < 0:
            _lib.check(int(need), "tree_verify_attention(workspace)")
        if need > 0:
            if self._ws is None or self._ws.numel() < need or self._ws.device != q.device:
                self._ws = torch.empty((int(need),), dtype=torch.uint8, device=q.device)
            a.workspace, a.workspace_bytes = self._ws.data_ptr(), self._ws.numel()
        rc = lib.sdb_tree_attn(a, _lib.stream_ptr(stream))
        _lib.check(rc, "tree_verify_attention")
        return out, lse


_default_launcher = TreeVerifyAttention()


def tree_verify_attention(*args, **kwargs):
    """Batched paged GQA tree attention (prefix + masked suffix + LSE merge).

    q bf16 [B, R, Hq, d]; k_cache/v_cache [num_blocks, Hkv, block_size, d];
    block_table int32 [B, max_blocks]; ctx_len int32 [B]; tree_k/v
    [B, R, Hkv, d]; mask_words int32 [B, R, W] (from drafttree.tree_build);
    n_rows int32 [B].  Returns (out [B, R, Hq, d], lse fp32 [B, Hq, R])."""
    return _default_launcher(*args, **kwargs)


def draft_tree_attention(q, k_cache, v_cache, block_table, ctx_len, suffix_k, suffix_v, mask_words, n_rows, q_row0,
                         scale, out=None, lse=None, **kw):
    """One depth step of the draft stage's tree attention (engine.py:424-432,
    model.py:257-270 with ``suffix_mask_new`` / ``carry_kv``), batched.

    The realized draft nodes are rows [0, n_rows[b]) of ``suffix_k/v``
    [B, R, Hkv, d] (carried K/V of earlier depths followed by this depth's new
    nodes); the new nodes are rows [q_row0[b], n_rows[b]) of ``q`` [B, R, Hq,
    d].  ``mask_words`` is ``tree_build`` of the realized parent array (the
    engine's vis_rows).  Only rows >= q_row0 of out / lse are written.
    ``max_q_nodes`` (host int, >= max over b of n_rows - q_row0, e.g. the
    depth's node count of the tree shape) sizes the work plan to the new
    rows instead of R."""
    return _default_launcher(q, k_cache, v_cache, block_table, ctx_len, suffix_k, suffix_v, mask_words, n_rows,
                             scale, out=out, lse=lse, q_row0=q_row0, **kw)
