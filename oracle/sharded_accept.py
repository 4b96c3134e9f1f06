"""CPU restatement of the vocab-sharded stochastic acceptance protocol --
TEST INFRASTRUCTURE ONLY (never the product path).

``paper_2508_08192_b200/csrc/accept_sharded.cu`` splits the reference's
T > 0 acceptance (``sampling.py:87-202``: ``target_dist`` with top-p for every
tree row, the parent rows' draft q, ``mss_verify``) over vocabulary shards,
with one batched collective between phases (``sharding.run_sharded_stochastic``).
This module runs the SAME decomposition in float64 numpy for one sequence on
one rank, with the collectives supplied by the caller (``comm``), so that a
world_size > 1 gloo test on CPU can show the decomposition reproduces the
unsharded reference (``specdec_oracle.mss_verify``) on every rank:

  1. local (max, sum exp) per row -> all-gather -> global softmax stats
  2. exact top-p cut: four byte-wise 256-bin mass histograms over the
     probability key (fp32 logit order, -0 == +0) -> all-reduce SUM each;
     per-rank tie counts -> all-reduce SUM; per-rank (key, index) cut
  3. p(t), q(t) of every drafted token -> all-reduce SUM
  4. rejection chain (c_k, M_k) of every parent row, level by level
     (siblings share the parent q, engine.py:405-407) -> all-reduce SUM each
  5. identical walk on every rank; local bonus mass -> all-reduce SUM;
     the owning rank's inverse CDF -> all-reduce MAX
"""

from __future__ import annotations

import numpy as np


def prob_keys(logits_f32):
    """uint32 order key of fp32 logits (larger logit -> larger key, -0 == +0)."""
    x = np.where(logits_f32 == 0, np.float32(0.0), logits_f32).astype(np.float32)
    b = x.view(np.uint32).astype(np.uint64)
    return np.where(b & 0x80000000, (~b) & 0xFFFFFFFF, b | 0x80000000).astype(np.uint64)


def sharded_accept(comm, target, draft, v_lo, vocab, parent, tokens, uniforms, temperature, top_p):
    """One sequence on one rank.  target/draft: float32 (R, V_local) slices of
    the augmented tree rows (row 0 = root); parent: augmented parents (row 0 =
    -1); tokens: global token ids per row (row 0 unused).  Returns (path,
    next_token, uniforms_used) -- identical on every rank."""
    R, vl = target.shape
    inv_t = 1.0 / temperature
    children = [[j for j in range(R) if parent[j] == r] for r in range(R)]
    prow = [r for r in range(R) if children[r]]
    # 1. softmax stats: local (max, sum) -> all-gather
    loc = np.zeros((R, 2, 2))
    for r in range(R):
        for z, rows in enumerate((target, draft)):
            if z == 1 and not children[r]:
                loc[r, z] = (-np.inf, 0.0)
                continue
            x = rows[r].astype(np.float64) * inv_t
            m = x.max()
            loc[r, z] = (m, np.exp(x - m).sum())
    allp = comm.all_gather(loc)  # (G, R, 2, 2)
    M = allp[:, :, :, 0].max(axis=0)
    with np.errstate(invalid="ignore"):
        S = np.where(np.isfinite(allp[:, :, :, 0]), allp[:, :, :, 1] * np.exp(allp[:, :, :, 0] - M[None]), 0.0).sum(0)
    keys = prob_keys(target)
    w_t = np.exp(target.astype(np.float64) * inv_t - M[:, 0, None])  # unnormalised target weights
    keep = np.ones((R, vl), dtype=bool)
    Z = S[:, 0].copy()
    # 2. exact top-p cut (reference sort order: prob desc, index asc)
    if top_p < 1.0:
        tau = (top_p - 1e-12) * S[:, 0]
        prefix = np.zeros(R, dtype=np.uint64)
        above = np.zeros(R)
        for k in range(4):
            hi_shift, shift = 32 - 8 * k, 24 - 8 * k
            hist = np.zeros((R, 256))
            for r in range(R):
                sel = np.ones(vl, dtype=bool) if k == 0 else (keys[r] >> np.uint64(hi_shift)) == prefix[r]
                np.add.at(hist[r], ((keys[r][sel] >> np.uint64(shift)) & np.uint64(0xFF)).astype(np.int64),
                          w_t[r][sel])
            hist = comm.all_reduce_sum(hist)
            for r in range(R):
                cum = above[r]
                chosen, last_nz = None, None
                for b in range(255, -1, -1):
                    if hist[r, b] > 0:
                        last_nz = b
                        if cum + hist[r, b] >= tau[r]:
                            chosen = b
                            break
                    cum += hist[r, b]
                if chosen is None:  # rounding kept the total below tau: keep down to the lowest bin
                    chosen = last_nz if last_nz is not None else 0
                    cum -= hist[r, chosen] if last_nz is not None else 0.0
                prefix[r] = (prefix[r] << np.uint64(8)) | np.uint64(chosen)
                above[r] = cum
        ties = np.zeros((R, comm.world), dtype=np.int64)
        for r in range(R):
            ties[r, comm.rank] = int((keys[r] == prefix[r]).sum())
        ties = comm.all_reduce_sum(ties)
        for r in range(R):
            kf = np.array([prefix[r]], dtype=np.uint64)
            bits = np.where(kf & np.uint64(0x80000000), kf & np.uint64(0x7FFFFFFF), (~kf) & np.uint64(0xFFFFFFFF))
            l_cut = float(bits.astype(np.uint32).view(np.float32)[0])
            w = np.exp(l_cut * inv_t - M[r, 0])
            total = int(ties[r].sum())
            need = int(min(max(np.ceil((tau[r] - above[r]) / w), 1), total))
            before = int(ties[r, :comm.rank].sum())
            mine = int(ties[r, comm.rank])
            kl = min(max(need - before, 0), mine)
            tied = np.nonzero(keys[r] == prefix[r])[0]
            keep[r] = (keys[r] > prefix[r])
            keep[r, tied[:kl]] = True
            Z[r] = above[r] + w * need
    P = np.where(keep, w_t, 0.0) / Z[:, None]
    with np.errstate(invalid="ignore", over="ignore"):
        Q = np.exp(draft.astype(np.float64) * inv_t - M[:, 1, None]) / S[:, 1, None]
    # 3. p(t), q(t) of every drafted token (owner contributes)
    pq = np.zeros((R, 2))
    for j in range(1, R):
        t = int(tokens[j]) - v_lo
        if 0 <= t < vl:
            pq[j] = (P[parent[j], t], Q[parent[j], t])
    pq = comm.all_reduce_sum(pq)
    # 4. rejection chains of every parent row, level-synchronous
    levels = max((len(c) for c in children), default=0)
    chain = {r: [(0.0, 1.0)] for r in prow}
    for k in range(1, levels + 1):
        x = np.zeros(R)
        for r in prow:
            if len(children[r]) >= k:
                c, m = chain[r][k - 1]
                x[r] = np.maximum(P[r] - (c + m) * Q[r], 0.0).sum()
        x = comm.all_reduce_sum(x)
        for r in prow:
            if len(children[r]) >= k:
                c, m = chain[r][k - 1]
                chain[r].append((0.0, 1.0) if x[r] / m <= 1e-12 else (c + m, x[r]))
    # 5. the walk (identical on every rank), then the bonus draw
    cur, k, used, path = 0, 0, 0, []
    while True:
        descended = False
        for j in children[cur]:
            u = uniforms[used]
            used += 1
            p_t, q_t = pq[j]
            c, m = chain[cur][k]
            pt = max(p_t - c * q_t, 0.0) / m
            if (pt > 0.0) if q_t <= 0.0 else (u < min(1.0, pt / q_t)):
                path.append(j - 1)
                cur, k, descended = j, 0, True
                break
            k += 1
        if not descended:
            break
    u = uniforms[used]
    used += 1
    c, m = chain[cur][k] if cur in chain else (0.0, 1.0)
    p_fin = np.maximum(P[cur] - (c * Q[cur] if c != 0.0 else 0.0), 0.0) / m
    mass = np.zeros(comm.world)
    mass[comm.rank] = p_fin.sum()
    mass = comm.all_reduce_sum(mass)
    base = mass[:comm.rank].sum()
    tok = -1
    if base <= u < base + mass[comm.rank]:
        idx = int(np.searchsorted(base + np.cumsum(p_fin), u, side="right"))
        tok = v_lo + min(idx, vl - 1)
    elif comm.rank == comm.world - 1 and mass.sum() <= u:
        tok = vocab - 1
    tok = int(comm.all_reduce_max(np.array([tok]))[0])
    return path, tok, used
