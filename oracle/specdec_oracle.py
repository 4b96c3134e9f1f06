"""CPU oracle for the EAGLE tree-verification hot path -- TEST INFRASTRUCTURE ONLY.

This module is a numpy restatement of the reference package ``specdec``
(arXiv 2508.08192, /root/reference/pkg/src/specdec) for exactly the functions
on the tree-verify path.  It exists to CHECK the CUDA product path; it is
never the thing measured or shipped.  Only ``tests/``,
``__graft_entry__.smoke()`` and ``bench.py``'s ``cpu_baseline`` / ``--impl
reference`` leg may import it.

Parity pinning: every function here is checked against golden vectors that
``oracle/make_golden.py`` produced by importing the UNMODIFIED reference
(``tests/golden/*.npz``; see ``tests/test_oracle_golden.py``).  So the oracle
is pinned to the reference's own outputs, not just to its reading of the
source.

Conventions (reference file:line in each docstring):
  * float64 everywhere (``numcore.py:14``);
  * trees are parent tuples with ROOT = -1 and parent[i] < i
    (``drafttree.py:13, 26-35``);
  * "augmented" trees prepend the root token as node 0 (``engine.py:170-173``);
  * device K/V page layout is ``[num_blocks, n_kv_heads, block_size, head_dim]``
    (a (page, head) tile is contiguous); the reference's logical layout is
    token-major ``[block, slot, H*d]`` (``kvstore.py:122-123``).  Both give
    the same gathered rows; ``paged_gather`` below restates ``gather``.
"""

from __future__ import annotations

import numpy as np

ROOT = -1
NEG_INF = float("-inf")


class OracleError(ValueError):
    """Mirrors the reference's ValueError subclasses (TreeError, AttentionError,
    SamplingError) -- the oracle only needs to raise *something* on the same
    inputs the reference rejects."""


# ---------------------------------------------------------------------------
# K0: tree structure (drafttree.py / engine.py)
# ---------------------------------------------------------------------------

def tree_depth(parent):
    """Per-node depth; root children have depth 1.

    Restates ``TreeSpec.__post_init__`` (drafttree.py:26-35): parent must be
    ROOT or an earlier index, otherwise TreeError.
    """
    depth = []
    for i, p in enumerate(parent):
        if p == ROOT:
            depth.append(1)
        elif 0 <= p < i:
            depth.append(depth[p] + 1)
        else:
            raise OracleError(f"node {i}: parent {p} must precede it or be ROOT")
    return np.asarray(depth, dtype=np.int64)


def augment(parent):
    """Prepend the root (last committed token) as node 0 (engine.py:170-173)."""
    return (ROOT,) + tuple(0 if p == ROOT else p + 1 for p in parent)


def suffix_mask(parent):
    """Ancestor-or-self closure as an (n, n) bool matrix (drafttree.py:102-111)."""
    n = len(parent)
    mask = np.zeros((n, n), dtype=bool)
    for i in range(n):
        p = parent[i]
        if p != ROOT:
            mask[i] = mask[p]
        mask[i, i] = True
    return mask


def mask_words(mask, n_words=None):
    """Pack an (R, R) bool mask into uint32 words per row, LSB = column 0.

    This is the device layout of the K0 output."""
    r, c = mask.shape
    w = n_words if n_words is not None else max(1, -(-c // 32))
    out = np.zeros((r, w), dtype=np.uint32)
    for i in range(r):
        for j in np.nonzero(mask[i])[0]:
            out[i, j // 32] |= np.uint32(1) << np.uint32(j % 32)
    return out


def positions(parent, ctx_len):
    """Absolute query positions ``ctx + depth - 1``.

    ``tree_attention`` uses ``ctx + d - 1`` on the tree it is given
    (attention.py:142); the engine passes the augmented tree with
    ``L - 2 + depth_aug`` where ctx = L - 1 (engine.py:456, model.py:235), the
    same formula.
    """
    return ctx_len + tree_depth(parent) - 1


# ---------------------------------------------------------------------------
# K1-K3: attention (kernels.py / attention.py / kvstore.py)
# ---------------------------------------------------------------------------

def attend_heads(q, k, v, mask, scale):
    """Masked softmax(q k^T * scale) v with per-row natural-log LSE.

    Restates ``_attend_numpy`` (kernels.py:40-54): q (H, m, d), k/v (H, n, d),
    mask (m, n) bool or None.  Fully-masked rows -> out 0, lse -inf.
    """
    scores = np.matmul(q, np.swapaxes(k, 1, 2)) * scale
    if mask is not None:
        scores = np.where(mask[None, :, :], scores, NEG_INF)
    smax = np.max(scores, axis=-1)
    alive = np.isfinite(smax)
    safe_max = np.where(alive, smax, 0.0)
    with np.errstate(invalid="ignore"):
        w = np.exp(np.where(np.isfinite(scores), scores - safe_max[..., None], NEG_INF))
    denom = np.sum(w, axis=-1)
    safe_denom = np.where(denom > 0.0, denom, 1.0)
    out = np.matmul(w, v) / safe_denom[..., None]
    out = np.where(alive[..., None], out, 0.0)
    lse = np.where(alive, safe_max + np.log(safe_denom), NEG_INF)
    return out, lse


def attend(q, k, v, mask, scale, n_heads):
    """Row-matrix front end of ``attention.attend`` (attention.py:92-105).

    q (m, H*d), k/v (n, H*d); returns (out (m, H*d), lse (H, m)).  Empty keys
    give out 0 and lse -inf (attention.py:98-100)."""
    m, dim = q.shape
    n = k.shape[0]
    dh = dim // n_heads
    if n == 0:
        return np.zeros((m, dim)), np.full((n_heads, m), NEG_INF)
    split = lambda x: np.ascontiguousarray(x.reshape(x.shape[0], n_heads, dh).transpose(1, 0, 2))
    out, lse = attend_heads(split(q), split(k), split(v), mask, scale)
    return np.ascontiguousarray(out.transpose(1, 0, 2)).reshape(m, dim), lse


def merge_partials(parts, n_heads):
    """LSE merge of disjoint-key partials (attention.py:108-124).

    parts: list of (out (m, H*d), lse (H, m)).  Raises if a row is masked in
    every part."""
    if not parts:
        raise OracleError("merge: no parts")
    lses = np.stack([p[1] for p in parts])
    m_rows, dim = parts[0][0].shape
    dh = dim // n_heads
    outs = np.stack([p[0].reshape(m_rows, n_heads, dh).transpose(1, 0, 2) for p in parts])
    mx = np.max(lses, axis=0)
    if not np.isfinite(mx).all():
        raise OracleError("merge: query row masked in every part")
    w = np.exp(lses - mx[None])
    denom = np.sum(w, axis=0)
    merged = np.sum(w[..., None] * outs, axis=0) / denom[..., None]
    out = np.ascontiguousarray(merged.transpose(1, 0, 2)).reshape(m_rows, dim)
    return out, mx + np.log(denom)


def gqa_repeat(x, n_kv_heads, group):
    """GQA adapter: repeat each KV head ``group`` times so the reference's MHA
    attention serves q head h with kv head h // group (SURVEY.md section 0.4,
    8c)."""
    rows = x.shape[0]
    d = x.shape[1] // n_kv_heads
    return np.repeat(x.reshape(rows, n_kv_heads, d), group, axis=1).reshape(rows, n_kv_heads * group * d)


def tree_attention(q_tree, committed_k, committed_v, tree_k, tree_v, parent, scale,
                   n_heads, n_kv_heads=None, chunk_len=None):
    """Two-pass tree attention with LSE (attention.py:131-151 + 108-124).

    q_tree (R, Hq*d); committed_k/v (C, Hkv*d); tree_k/v (R, Hkv*d).  Returns
    (out (R, Hq*d), lse (Hq, R)).  ``chunk_len`` applies the iRoPE LocalChunk
    prefix mask (attention.py:33-40, 76-84).
    """
    n_kv = n_heads if n_kv_heads is None else n_kv_heads
    g = n_heads // n_kv
    ck, cv = gqa_repeat(committed_k, n_kv, g), gqa_repeat(committed_v, n_kv, g)
    tk, tv = gqa_repeat(tree_k, n_kv, g), gqa_repeat(tree_v, n_kv, g)
    ctx = ck.shape[0]
    depth = tree_depth(parent)
    parts = []
    if ctx > 0:
        pmask = None
        if chunk_len is not None:
            qp = ctx + depth - 1
            kp = np.arange(ctx)
            pmask = (qp[:, None] // chunk_len == kp[None, :] // chunk_len) & (kp[None, :] <= qp[:, None])
        parts.append(attend(q_tree, ck, cv, pmask, scale, n_heads))
    parts.append(attend(q_tree, tk, tv, suffix_mask(parent), scale, n_heads))
    return merge_partials(parts, n_heads)


def paged_gather(pool, block_table, n_rows):
    """Gather the first n committed rows of one sequence from a paged pool.

    Restates ``PagedKvCache.gather`` / ``_segments`` (kvstore.py:207-215,
    235-246) -- one copy per page segment -- on the device layout
    pool[num_blocks, Hkv, bs, d]; returns (n, Hkv*d) rows."""
    nb, hkv, bs, d = pool.shape
    segs = []
    pos = 0
    while pos < n_rows:
        b, off = divmod(pos, bs)
        take = min(bs - off, n_rows - pos)
        seg = pool[block_table[b], :, off:off + take, :]  # (hkv, take, d)
        segs.append(np.transpose(seg, (1, 0, 2)).reshape(take, hkv * d))
        pos += take
    if not segs:
        return np.zeros((0, hkv * d), dtype=pool.dtype)
    return np.concatenate(segs)


def paged_write(pool, block_table, start, rows):
    """Write rows (n, Hkv*d) at positions start.. of one sequence.

    Restates ``PagedKvCache.write`` (kvstore.py:217-225)."""
    nb, hkv, bs, d = pool.shape
    for i in range(rows.shape[0]):
        b, off = divmod(start + i, bs)
        pool[block_table[b], :, off, :] = rows[i].reshape(hkv, d)


def tree_verify_attention_batch(q, k_pool, v_pool, block_table, ctx_len, tree_k, tree_v,
                                parents, scale, chunk_len=None):
    """Batched oracle of the device op ``tree_verify_attn``.

    q (B, R, Hq, d); pools (nb, Hkv, bs, d); tree_k/v (B, R, Hkv, d);
    parents: list of per-sequence parent tuples (length n_rows[b] <= R).
    Returns out (B, R, Hq, d) and lse (B, Hq, R) (padding rows 0 / -inf).
    Loops sequences one after another like the engine (engine.py:581-582).
    """
    bsz, r_max, hq, d = q.shape
    hkv = k_pool.shape[1]
    out = np.zeros((bsz, r_max, hq, d))
    lse = np.full((bsz, hq, r_max), NEG_INF)
    for b in range(bsz):
        n = len(parents[b])
        c = int(ctx_len[b])
        ck = paged_gather(k_pool, block_table[b], c)
        cv = paged_gather(v_pool, block_table[b], c)
        o, l = tree_attention(q[b, :n].reshape(n, hq * d), ck, cv,
                              tree_k[b, :n].reshape(n, hkv * d), tree_v[b, :n].reshape(n, hkv * d),
                              parents[b], scale, hq, hkv, chunk_len)
        out[b, :n] = o.reshape(n, hq, d)
        lse[b, :, :n] = l
    return out, lse


def draft_depth_attention(q_new, committed_k, committed_v, suffix_k, suffix_v, mask_new, scale, n_heads,
                          n_kv_heads=None):
    """One depth step of the draft stage's tree attention (engine.py:424-432
    -> model.py:257-270 with ``suffix_mask_new`` and ``carry_kv``): the new
    nodes' queries attend the draft cache prefix (CausalPrefix: every
    committed key) plus the suffix = carried K/V of the earlier nodes ++ the
    new nodes' K/V under the rectangular visibility ``mask_new`` (n_new,
    total), merged by LSE.  q_new (n_new, Hq*d); suffix_k/v (total, Hkv*d).
    Returns (out (n_new, Hq*d), lse (Hq, n_new))."""
    n_kv = n_heads if n_kv_heads is None else n_kv_heads
    g = n_heads // n_kv
    ck, cv = gqa_repeat(committed_k, n_kv, g), gqa_repeat(committed_v, n_kv, g)
    sk, sv = gqa_repeat(suffix_k, n_kv, g), gqa_repeat(suffix_v, n_kv, g)
    parts = []
    if ck.shape[0] > 0:
        parts.append(attend(q_new, ck, cv, None, scale, n_heads))
    parts.append(attend(q_new, sk, sv, np.asarray(mask_new, dtype=bool), scale, n_heads))
    return merge_partials(parts, n_heads)


def draft_depth_attention_batch(q, k_pool, v_pool, block_table, ctx_len, suffix_k, suffix_v, parents, q_row0,
                                scale):
    """Batched oracle of the rectangular device call (``q_row0``): rows
    [q_row0[b], len(parents[b])) of q (B, R, Hq, d) attend; suffix keys are
    all realized nodes [0, len(parents[b])) with the ancestor-or-self mask of
    the realized draft tree (engine.py:409-421 vis_rows).  Returns out / lse
    arrays with only those rows filled (others NaN)."""
    bsz, r_max, hq, d = q.shape
    hkv = k_pool.shape[1]
    out = np.full((bsz, r_max, hq, d), np.nan)
    lse = np.full((bsz, hq, r_max), np.nan)
    for b in range(bsz):
        n, q0 = len(parents[b]), int(q_row0[b])
        if q0 >= n:
            continue
        c = int(ctx_len[b])
        ck = paged_gather(k_pool, block_table[b], c)
        cv = paged_gather(v_pool, block_table[b], c)
        mask = suffix_mask(parents[b])[q0:n]
        o, l = draft_depth_attention(q[b, q0:n].reshape(n - q0, hq * d), ck, cv,
                                     suffix_k[b, :n].reshape(n, hkv * d), suffix_v[b, :n].reshape(n, hkv * d),
                                     mask, scale, hq, hkv)
        out[b, q0:n] = o.reshape(n - q0, hq, d)
        lse[b, :, q0:n] = l
    return out, lse


# ---------------------------------------------------------------------------
# K4-K6: target distribution, acceptance, uniforms (numcore.py / sampling.py)
# ---------------------------------------------------------------------------

def softmax_lse(logits, temperature):
    """Row softmax of logits/T; T == 0 -> one-hot argmax, lowest index on ties.

    Restates numcore.py:41-60 (NaN -> error)."""
    logits = np.asarray(logits, dtype=np.float64)
    if np.isnan(logits).any():
        raise OracleError("softmax_lse: NaN in logits")
    if temperature < 0:
        raise OracleError("softmax_lse: negative temperature")
    if temperature == 0:
        probs = np.zeros_like(logits)
        idx = np.argmax(logits, axis=1)
        probs[np.arange(logits.shape[0]), idx] = 1.0
        return probs, logits[np.arange(logits.shape[0]), idx].copy()
    scaled = logits / temperature
    m = np.max(scaled, axis=1, keepdims=True)
    lse = m[:, 0] + np.log(np.sum(np.exp(scaled - m), axis=1))
    return np.exp(scaled - lse[:, None]), lse


def check_dist(dist):
    """sampling.py:43-49."""
    d = np.asarray(dist, dtype=np.float64)
    if d.ndim != 1:
        raise OracleError("distribution must be 1-D")
    if (d < 0).any() or abs(float(d.sum()) - 1.0) > 1e-9:
        raise OracleError("distribution entries must be >= 0 and sum to 1")
    return d


def top_p_mask(dist, p):
    """Smallest (prob desc, index asc) prefix with mass >= p, renormalised.

    Restates sampling.py:52-72 (cutoff = searchsorted(cumsum, p - 1e-12))."""
    d = check_dist(dist)
    if not 0 < p <= 1:
        raise OracleError("top_p must be in (0, 1]")
    order = np.lexsort((np.arange(d.shape[0]), -d))
    csum = np.cumsum(d[order])
    cutoff = min(int(np.searchsorted(csum, p - 1e-12)), d.shape[0] - 1)
    keep = order[:cutoff + 1]
    out = np.zeros_like(d)
    out[keep] = d[keep]
    return out / out.sum()


def target_dist(logits_row, temperature, top_p, allowed=None):
    """Logits row -> sampling distribution: FSM mask, temperature, top-p.

    Restates sampling.py:87-102."""
    row = np.asarray(logits_row, dtype=np.float64)
    if allowed is not None:
        if not allowed.any():
            raise OracleError("no token allowed (dead FSM state)")
        row = np.where(allowed, row, -np.inf)
    d = softmax_lse(row[None, :], temperature)[0][0]
    if top_p < 1:
        d = top_p_mask(d, top_p)
    return d


def sample_from(dist, u):
    """Inverse-CDF draw (sampling.py:105-109)."""
    d = check_dist(dist)
    idx = int(np.searchsorted(np.cumsum(d), u, side="right"))
    return min(idx, d.shape[0] - 1)


def children(parent, i):
    """Children of node i (or ROOT) in priority (= index) order (drafttree.py:45-47)."""
    return [j for j, p in enumerate(parent) if p == i]


def mss_verify(parent, node_tokens, node_dists, target_dists, uniforms):
    """Multi-round speculative sampling tree walk (sampling.py:149-202).

    parent: NON-augmented draft tree; node_dists[c] is the draft q that
    proposed node c; target_dists[0] is the root context, [1+i] node i's.
    Returns (accepted_path, next_token, residual, uniforms_used).

    Test-size shortcut: node_dists / target_dists may also be callables
    (index -> dist), evaluated and checked only for the rows the walk reads
    (the reference checks every row first; the walk itself is identical).
    Used at the full Llama-3 vocabulary for batches of 64 sequences, where
    the top-p sort of every row would take minutes."""
    if callable(target_dists):
        memo = {}

        def tdist(i):
            if i not in memo:
                memo[i] = check_dist(target_dists(i))
            return memo[i]
    else:
        if len(target_dists) != len(parent) + 1:
            raise OracleError("need one target dist per node parent incl. root")
        dists = [check_dist(d) for d in target_dists]
        tdist = dists.__getitem__
    qdist = node_dists if callable(node_dists) else node_dists.__getitem__
    used = 0
    cur = ROOT
    p = tdist(0)
    anchor = p
    path = []
    while True:
        descended = False
        for c in children(parent, cur):
            t = node_tokens[c]
            q = qdist(c)
            if used >= len(uniforms):
                raise OracleError("uniform stream exhausted mid-walk")
            u = uniforms[used]
            used += 1
            qt, pt = float(q[t]), float(p[t])
            accept = (pt > 0.0) if qt <= 0.0 else (u < min(1.0, pt / qt))
            if accept:
                path.append(c)
                p = tdist(1 + c)
                anchor = p
                cur = c
                descended = True
                break
            residual = np.maximum(p - q, 0.0)
            mass = float(residual.sum())
            p = anchor if mass <= 1e-12 else residual / mass
        if not descended:
            break
    if used >= len(uniforms):
        raise OracleError("uniform stream exhausted before bonus draw")
    token = sample_from(p, uniforms[used])
    used += 1
    return path, token, p, used


def greedy_walk(parent, node_tokens, argmax_rows):
    """Temperature-0 acceptance as an argmax walk.

    Equivalent to ``mss_verify`` with one-hot target dists
    (numcore.py:51-55): at node `cur` the child whose token equals the argmax
    of row (1+cur) is accepted (first such child in priority order); every
    other examined child is rejected -- its p(t) is 0 -- and the residual of a
    one-hot p minus any q stays that one-hot (or the anchor, the same one-hot).
    The bonus is argmax at the stop node.  uniforms_used counts candidates
    examined + 1, exactly as mss_verify consumes them.  Pinned against the
    real mss_verify by tests/golden/accept_greedy.npz.
    argmax_rows[0] is the root row, argmax_rows[1+i] node i's row."""
    cur = ROOT
    used = 0
    path = []
    while True:
        want = int(argmax_rows[0 if cur == ROOT else 1 + cur])
        nxt = None
        for c in children(parent, cur):
            used += 1
            if int(node_tokens[c]) == want:
                nxt = c
                break
        if nxt is None:
            break
        path.append(nxt)
        cur = nxt
    bonus = int(argmax_rows[0 if cur == ROOT else 1 + cur])
    return path, bonus, used + 1


# Philox4x64-10 as numpy's BitGenerator runs it (sampling.py:112-124 uses
# np.random.Philox(key=(seed, step))): counter pre-incremented, so element i of
# the row-major (rows, width) matrix is lane i % 4 of block counter i // 4 + 1,
# mapped to a double as (x >> 11) * 2**-53.
_PM0, _PM1 = 0xD2E7470EE14C6C93, 0xCA5A826395121157
_PW0, _PW1 = 0x9E3779B97F4A7C15, 0xBB67AE8584CAA73B
_M64 = (1 << 64) - 1


def philox4x64_10(counter, key):
    c0, c1, c2, c3 = counter
    k0, k1 = key
    for _ in range(10):
        p0 = _PM0 * c0
        p1 = _PM1 * c2
        hi0, lo0 = p0 >> 64, p0 & _M64
        hi1, lo1 = p1 >> 64, p1 & _M64
        c0, c1, c2, c3 = (hi1 ^ c1 ^ k0) & _M64, lo1, (hi0 ^ c3 ^ k1) & _M64, lo0
        k0, k1 = (k0 + _PW0) & _M64, (k1 + _PW1) & _M64
    return c0, c1, c2, c3


def rank_sliced_uniforms(seed, step, padded_batch, row_width):
    """Full (padded_batch, row_width) uniform matrix for one step, restating
    ``rank_sliced_uniforms`` (sampling.py:112-124) with an explicit
    Philox4x64-10 (so a device Philox can be written against it)."""
    if padded_batch < 1 or row_width < 0:
        raise OracleError("padded_batch must be >= 1 and row_width >= 0")
    n = padded_batch * row_width
    out = np.empty(n, dtype=np.float64)
    key = (seed & _M64, step & _M64)
    for blk in range(-(-n // 4)):
        words = philox4x64_10((blk + 1, 0, 0, 0), key)
        for lane in range(4):
            i = blk * 4 + lane
            if i < n:
                out[i] = (words[lane] >> 11) * (1.0 / 9007199254740992.0)
    return out.reshape(padded_batch, row_width)


def uniform_row(seed, step, width, batch_size=1, world=1):
    """Row 0 of the padded Philox matrix (engine.py:251-254)."""
    padded = -(-batch_size // world) * world
    return rank_sliced_uniforms(seed, step, padded, width)[0]


# ---------------------------------------------------------------------------
# K7: compaction of the accepted path (engine.py:504-523)
# ---------------------------------------------------------------------------

def accepted_rows(path, n_keep):
    """Tree rows written back: root + accepted nodes except the last kept
    token's (engine.py:514-517)."""
    write_path = list(path)[:n_keep - 1]
    return [0] + [1 + a for a in write_path]


def compact_kv(k_pool, v_pool, block_table, ctx_len, tree_k, tree_v, path, n_keep):
    """Write the accepted rows of one sequence/layer into its pages at
    positions ctx_len .. (engine.py:518-520 -> kvstore.py:217-225; ctx = L-1).

    tree_k/v (R, Hkv, d) in augmented row order.  Modifies pools in place."""
    rows = accepted_rows(path, n_keep)
    r = np.asarray(rows)
    hkv, d = tree_k.shape[1], tree_k.shape[2]
    paged_write(k_pool, block_table, ctx_len, tree_k[r].reshape(len(rows), hkv * d))
    paged_write(v_pool, block_table, ctx_len, tree_v[r].reshape(len(rows), hkv * d))
    return rows


# ---------------------------------------------------------------------------
# Bookkeeping either side of the step (engine.py:504-533), logical view
# ---------------------------------------------------------------------------

def bookkeep_round(base_rows, draft_rows, tape_rows, L, path, kept, base_kv, suffix_kv, hidden, align_kv):
    """One round of the engine's bookkeeping on logical (position-indexed)
    rows, restating engine.py:514-533 + PagedKvCache.write / rewind / set_len
    (kvstore.py:217-225, 248-258) and HiddenTape.append_rows (405-409).

    base_rows / draft_rows: per layer [k_rows, v_rows] lists (committed
    positions 0 .. L-2); tape_rows: list of hidden rows.  The draft's
    alignment write (align_kv per layer, position L-1) precedes the
    write-back.  Returns the new committed length."""
    write_path = list(path)[:kept - 1]
    rows = accepted_rows(path, kept)
    new_len = L + kept
    for li, (k, v) in enumerate(base_kv):
        for j, rr in enumerate(rows):
            for col, src in ((0, k), (1, v)):
                seq = base_rows[li][col]
                pos = L - 1 + j
                if pos < len(seq):
                    seq[pos] = src[rr]
                else:
                    seq.append(src[rr])
        for col in (0, 1):
            del base_rows[li][col][new_len - 1:]
    for li, (k, v) in enumerate(suffix_kv):
        for col, src in ((0, k), (1, v)):
            seq = draft_rows[li][col]
            a = align_kv[li][col]
            if L - 1 < len(seq):
                seq[L - 1] = a
            else:
                seq.append(a)
            for j, node in enumerate(write_path):
                pos = L + j
                if pos < len(seq):
                    seq[pos] = src[node]
                else:
                    seq.append(src[node])
            del seq[new_len - 1:]
    tape_rows.extend([hidden[0]] + [hidden[1 + a] for a in write_path])
    return new_len
