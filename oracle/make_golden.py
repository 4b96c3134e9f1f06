"""Generate golden fixtures by running the UNMODIFIED reference ``specdec``.

TEST INFRASTRUCTURE.  Run in the dev container only (the reference is not on
the GPU box):

    PYTHONDONTWRITEBYTECODE=1 NUMBA_CACHE_DIR=/tmp/numba_cache \
        python oracle/make_golden.py

It imports /root/reference/pkg/src/specdec read-only, drives the reference's
own public functions on seeded inputs and writes ``tests/golden/*.npz``.  The
fixtures pin both the oracle (tests/test_oracle_golden.py, CPU) and the CUDA
path (tests/test_gpu_*.py) to the reference's outputs.
"""

import os
import sys

import numpy as np

REF_SRC = "/root/reference/pkg/src"
OUT = os.path.join(os.path.dirname(os.path.abspath(__file__)), "..", "tests", "golden")

sys.path.insert(0, REF_SRC)
os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/numba_cache")

from specdec import attention as R_att  # noqa: E402
from specdec import drafttree as R_tree  # noqa: E402
from specdec import engine as R_eng  # noqa: E402
from specdec import kvstore as R_kv  # noqa: E402
from specdec import sampling as R_smp  # noqa: E402

# The 63-node EAGLE-style tree of SURVEY.md section 8(d) (R = 64 rows with root).
TREE64 = ("nodes:[-1,-1,-1,-1,-1,-1,-1,-1,0,0,0,0,0,0,1,1,1,1,1,2,2,2,2,3,3,3,4,4,5,5,6,7,"
          "8,8,8,8,9,9,9,10,10,10,11,11,12,13,14,15,32,32,32,33,33,34,34,35,36,37,48,48,49,"
          "50,51]")
TREE65 = TREE64[:-1] + ",0]"
N8 = "nodes:[-1,-1,0,0,1,2,2,5]"


def bf16_round(x):
    """Round float64 -> bf16 (round-to-nearest-even) -> float64."""
    f = np.asarray(x, dtype=np.float32)
    u = f.view(np.uint32).astype(np.uint64)
    u = ((u + 0x7FFF + ((u >> 16) & 1)) >> 16) << 16
    return u.astype(np.uint32).view(np.float32).astype(np.float64)


def random_tree(rng, n, p_root=0.2):
    parent = []
    for i in range(n):
        if i == 0 or rng.random() < p_root:
            parent.append(-1)
        else:
            parent.append(int(rng.integers(0, i)))
    return tuple(parent)


def pad_parents(parents, width):
    out = np.full((len(parents), width), -2, dtype=np.int32)
    lens = np.zeros(len(parents), dtype=np.int32)
    for i, p in enumerate(parents):
        out[i, :len(p)] = p
        lens[i] = len(p)
    return out, lens


# ---------------------------------------------------------------------------
def gen_trees():
    rng = np.random.default_rng(101)
    specs = ["full:2,2", N8, TREE64, TREE65, "chain:3", "chain:1", "full:3,2"]
    trees = [R_tree.parse_tree(s) for s in specs] + [R_tree.EMPTY_TREE]
    trees += [R_tree.TreeSpec(random_tree(rng, int(rng.integers(1, 100)))) for _ in range(24)]
    aug = [R_eng._augment(t) for t in trees]
    width = max(a.n_nodes for a in aug)
    par, lens = pad_parents([a.parent for a in aug], width)
    raw, raw_lens = pad_parents([t.parent for t in trees], width)
    masks = np.zeros((len(aug), width, width), dtype=bool)
    depth = np.zeros((len(aug), width), dtype=np.int32)
    pos = np.zeros((len(aug), width), dtype=np.int64)
    ctx = rng.integers(0, 5000, size=len(aug)).astype(np.int64)
    for i, a in enumerate(aug):
        n = a.n_nodes
        masks[i, :n, :n] = R_tree.suffix_mask(a)
        depth[i, :n] = a.depth
        # engine.py:456 positions L-2+depth with ctx = L-1
        L = ctx[i] + 1
        pos[i, :n] = [L - 2 + d for d in a.depth]
    # invalid parent arrays the reference rejects (drafttree.py:31-34)
    bad = [(-1, 2, 1), (0,), (-1, -1, 5), (-1, 0, 2), (-3,)]
    bad_ok = []
    for b in bad:
        try:
            R_tree.TreeSpec(b)
            bad_ok.append(True)
        except R_tree.TreeError:
            bad_ok.append(False)
    badp, badl = pad_parents(bad, 4)
    np.savez_compressed(os.path.join(OUT, "trees.npz"), specs=np.array(specs + ["empty"] + ["random"] * 24),
                        raw_parent=raw, raw_len=raw_lens, parent_aug=par, n_rows=lens, mask=masks,
                        depth=depth, ctx=ctx, pos=pos, bad_parent=badp, bad_len=badl,
                        bad_valid=np.array(bad_ok))


# ---------------------------------------------------------------------------
def gen_attention_f64():
    """Reference's own randomized tree-attention suite shape
    (verify.py:255-285 / tests/test_attention.py:88-111), with outputs."""
    rng = np.random.default_rng(303)
    cases = {}
    for ci in range(60):
        n_heads = int(rng.choice([1, 2, 4]))
        head_dim = int(rng.choice([4, 8]))
        dim = n_heads * head_dim
        n_nodes = int(rng.integers(1, 17))
        ctx = int(rng.integers(0, 65))
        chunk = [None, 4, 8][int(rng.integers(3))]
        parent = tuple(int(rng.integers(-1, i)) for i in range(n_nodes))
        tree = R_tree.TreeSpec(parent)
        q = rng.normal(size=(n_nodes, dim))
        tk = rng.normal(size=(n_nodes, dim))
        tv = rng.normal(size=(n_nodes, dim))
        ck = rng.normal(size=(ctx, dim))
        cv = rng.normal(size=(ctx, dim))
        scale = head_dim ** -0.5
        out = R_att.tree_attention(q, ck, cv, tk, tv, tree, scale, n_heads=n_heads, chunk_len=chunk)
        # LSE through the reference merge of the same two parts
        parts = []
        q_pos = tuple(ctx + d - 1 for d in tree.depth)
        if ctx > 0:
            bias = R_att.CausalPrefix(ctx) if chunk is None else R_att.LocalChunk(chunk, q_pos, tuple(range(ctx)))
            parts.append(R_att.attend(q, ck, cv, bias, scale, n_heads))
        parts.append(R_att.attend(q, tk, tv, R_att.TreeSuffix(R_tree.suffix_mask(tree)), scale, n_heads))
        merged = R_att.merge_partials(parts, n_heads)
        assert np.max(np.abs(merged.out - out)) == 0.0
        pre = f"c{ci}_"
        cases[pre + "meta"] = np.array([n_heads, head_dim, ctx, -1 if chunk is None else chunk])
        cases[pre + "parent"] = np.array(parent, dtype=np.int64)
        for name, arr in (("q", q), ("tk", tk), ("tv", tv), ("ck", ck), ("cv", cv),
                          ("out", out), ("lse", merged.lse)):
            cases[pre + name] = arr
    cases["n_cases"] = np.array(60)
    np.savez_compressed(os.path.join(OUT, "attention_f64.npz"), **cases)

    # attend / merge known cases (tests/test_attention.py:22-85 shapes)
    rng = np.random.default_rng(2)
    q = rng.normal(size=(4, 8))
    k, v = rng.normal(size=(10, 8)), rng.normal(size=(10, 8))
    a = R_att.attend(q, k[:3], v[:3], R_att.CausalPrefix(3), 0.3, n_heads=2)
    b = R_att.attend(q, k[3:], v[3:], R_att.CausalPrefix(7), 0.3, n_heads=2)
    m = R_att.merge_partials([a, b], n_heads=2)
    e = R_att.attend(q, np.zeros((0, 8)), np.zeros((0, 8)), R_att.CausalPrefix(0), 0.3, n_heads=2)
    mask = rng.random((4, 10)) < 0.5
    mask[1] = False  # fully masked row
    c = R_att.attend(q, k, v, R_att.TreeSuffix(mask), 0.3, n_heads=2)
    np.savez_compressed(os.path.join(OUT, "attend_merge.npz"), q=q, k=k, v=v, a_out=a.out, a_lse=a.lse,
                        b_out=b.out, b_lse=b.lse, m_out=m.out, m_lse=m.lse, e_out=e.out, e_lse=e.lse,
                        mask=mask, c_out=c.out, c_lse=c.lse)


# ---------------------------------------------------------------------------
def _ref_gqa_tree_attention(q, ck, cv, tk, tv, tree, scale, hq, hkv):
    g = hq // hkv

    def rep(x):
        rows = x.shape[0]
        d = x.shape[1] // hkv
        return np.repeat(x.reshape(rows, hkv, d), g, axis=1).reshape(rows, hq * d)

    parts = []
    if ck.shape[0] > 0:
        parts.append(R_att.attend(q, rep(ck), rep(cv), R_att.CausalPrefix(ck.shape[0]), scale, hq))
    parts.append(R_att.attend(q, rep(tk), rep(tv), R_att.TreeSuffix(R_tree.suffix_mask(tree)), scale, hq))
    m = R_att.merge_partials(parts, hq)
    return m.out, m.lse


def gen_attention_gqa():
    """Batched paged GQA cases for the device op (bf16-rounded inputs)."""
    cases = [
        # name, B, Hq, Hkv, d, trees(spec per seq), ctx per seq, block_size
        ("c1", 1, 4, 1, 64, ["full:2,2"], [256], 16),
        ("c1n8", 1, 4, 1, 64, [N8], [256], 16),
        ("gqa_ragged", 3, 8, 2, 128, [TREE64, N8, "chain:3"], [300, 129, 1], 16),
        ("gqa_r65", 2, 16, 2, 128, [TREE65, "full:2,2"], [200, 64], 64),
        ("ctx0", 2, 8, 2, 128, ["chain:3", "empty"], [0, 77], 16),
    ]
    rng = np.random.default_rng(7)
    store = {}
    for name, bsz, hq, hkv, d, specs, ctxs, bs in cases:
        trees = [R_tree.EMPTY_TREE if s == "empty" else R_tree.parse_tree(s) for s in specs]
        aug = [R_eng._augment(t) for t in trees]
        r_max = max(a.n_nodes for a in aug)
        n_pages = [-(-c // bs) for c in ctxs]
        max_blocks = max(max(n_pages), 1)
        nb = sum(n_pages) + 3
        perm = rng.permutation(nb)
        table = np.full((bsz, max_blocks), 0, dtype=np.int32)
        k_pool = bf16_round(rng.normal(size=(nb, hkv, bs, d)))
        v_pool = bf16_round(rng.normal(size=(nb, hkv, bs, d)))
        cur = 0
        for b in range(bsz):
            for j in range(n_pages[b]):
                table[b, j] = perm[cur]
                cur += 1
        q = np.zeros((bsz, r_max, hq, d))
        tk = np.zeros((bsz, r_max, hkv, d))
        tv = np.zeros((bsz, r_max, hkv, d))
        out = np.zeros((bsz, r_max, hq, d))
        lse = np.full((bsz, hq, r_max), -np.inf)
        scale = d ** -0.5
        for b in range(bsz):
            n = aug[b].n_nodes
            q[b, :n] = bf16_round(rng.normal(size=(n, hq, d)))
            tk[b, :n] = bf16_round(rng.normal(size=(n, hkv, d)))
            tv[b, :n] = bf16_round(rng.normal(size=(n, hkv, d)))
            # reference paged cache holding the same committed rows
            cache = R_kv.PagedKvCache(1, hkv * d, n_blocks=nb, block_size=bs)
            cache.new_seq(0)
            c = ctxs[b]
            rows_k = np.zeros((c, hkv * d))
            rows_v = np.zeros((c, hkv * d))
            for pos in range(c):
                pg, off = divmod(pos, bs)
                rows_k[pos] = k_pool[table[b, pg], :, off, :].reshape(-1)
                rows_v[pos] = v_pool[table[b, pg], :, off, :].reshape(-1)
            cache.ensure(0, max(c, 1))
            if c:
                cache.write(0, 0, 0, rows_k, rows_v)
            ck, cv = cache.gather(0, 0, c)
            o, l = _ref_gqa_tree_attention(q[b, :n].reshape(n, -1), ck, cv, tk[b, :n].reshape(n, -1),
                                          tv[b, :n].reshape(n, -1), aug[b], scale, hq, hkv)
            out[b, :n] = o.reshape(n, hq, d)
            lse[b, :, :n] = l
        par, lens = pad_parents([a.parent for a in aug], r_max)
        pre = name + "_"
        store[pre + "meta"] = np.array([bsz, hq, hkv, d, bs, r_max])
        store[pre + "q"] = q.astype(np.float32)
        store[pre + "tk"] = tk.astype(np.float32)
        store[pre + "tv"] = tv.astype(np.float32)
        store[pre + "k_pool"] = k_pool.astype(np.float32)
        store[pre + "v_pool"] = v_pool.astype(np.float32)
        store[pre + "table"] = table
        store[pre + "ctx"] = np.array(ctxs, dtype=np.int32)
        store[pre + "parent_aug"] = par
        store[pre + "n_rows"] = lens
        store[pre + "out"] = out
        store[pre + "lse"] = lse
    store["names"] = np.array([c[0] for c in cases])
    np.savez_compressed(os.path.join(OUT, "attention_gqa.npz"), **store)


# ---------------------------------------------------------------------------
def _draft_tokens_greedy(rng, tree, target_logits):
    # tokens: the parent row's argmax with prob 0.6, else random
    toks = []
    V = target_logits.shape[1]
    for i, p in enumerate(tree.parent):
        row = 0 if p == -1 else 1 + p
        if rng.random() < 0.6:
            toks.append(int(np.argmax(target_logits[row])))
        else:
            toks.append(int(rng.integers(0, V)))
    return toks


def gen_accept():
    rng = np.random.default_rng(55)
    specs = ["full:2,2", N8, TREE64, "chain:3", "chain:1", "empty"]
    # greedy (T = 0), logits with forced ties
    g = {}
    k = 0
    for rep in range(4):
        for s in specs:
            tree = R_tree.EMPTY_TREE if s == "empty" else R_tree.parse_tree(s)
            n = tree.n_nodes
            V = [64, 1000, 4096, 4099][rep]
            if rep % 2 == 0:
                logits = rng.integers(-3, 4, size=(n + 1, V)).astype(np.float32)
            else:
                logits = (2.0 * rng.normal(size=(n + 1, V))).astype(np.float32)
            draft_logits = (logits + 0.5 * rng.normal(size=logits.shape)).astype(np.float32)
            toks = _draft_tokens_greedy(rng, tree, logits)
            dists = [R_smp.target_dist(logits[i], 0.0, 1.0) for i in range(n + 1)]
            qd = [R_smp.target_dist(draft_logits[0 if p == -1 else 1 + p], 0.0, 1.0) for p in tree.parent]
            seed = int(rng.integers(0, 2**31))
            uni = R_smp.rank_sliced_uniforms(seed, 2, 1, n + 1)[0]
            res = R_smp.mss_verify(R_smp.DraftResult(tree, tuple(toks), tuple(qd)), dists, uni,
                                   mode="greedy_children")
            pre = f"g{k}_"
            g[pre + "parent"] = np.array(tree.parent, dtype=np.int32)
            g[pre + "logits"] = logits
            g[pre + "tokens"] = np.array(toks, dtype=np.int32)
            g[pre + "path"] = np.array(res.accepted_path, dtype=np.int32)
            g[pre + "next"] = np.array(res.next_token)
            g[pre + "used"] = np.array(res.uniforms_used)
            k += 1
    g["n_cases"] = np.array(k)
    np.savez_compressed(os.path.join(OUT, "accept_greedy.npz"), **g)

    # stochastic: draft q from draft logits (top-p skipped, engine.py:266-269),
    # tokens sampled from q with the reference Philox draws (engine.py:368, 393-394)
    st = {}
    k = 0
    for temp, top_p in ((1.0, 1.0), (1.0, 0.9), (0.7, 0.95), (1.3, 0.8)):
        for s in ["full:2,2", N8, TREE64, "chain:3", "empty"]:
            tree = R_tree.EMPTY_TREE if s == "empty" else R_tree.parse_tree(s)
            n = tree.n_nodes
            V = 2048
            logits = (2.0 * rng.normal(size=(n + 1, V))).astype(np.float32)
            draft_logits = (logits + 0.5 * rng.normal(size=logits.shape)).astype(np.float32)
            seed = int(rng.integers(0, 2**31))
            draws = R_smp.rank_sliced_uniforms(seed, 1, 1, max(n, 1))[0]
            qd, toks = [], []
            for i, p in enumerate(tree.parent):
                q = R_smp.target_dist(draft_logits[0 if p == -1 else 1 + p], temp, 1.0)
                qd.append(q)
                toks.append(R_smp.sample_from(q, draws[i]))
            dists = [R_smp.target_dist(logits[i], temp, top_p) for i in range(n + 1)]
            uni = R_smp.rank_sliced_uniforms(seed, 2, 1, n + 1)[0]
            res = R_smp.mss_verify(R_smp.DraftResult(tree, tuple(toks), tuple(qd)), dists, uni,
                                   mode="stochastic")
            pre = f"s{k}_"
            st[pre + "meta"] = np.array([temp, top_p, seed])
            st[pre + "parent"] = np.array(tree.parent, dtype=np.int32)
            st[pre + "logits"] = logits
            st[pre + "draft_logits"] = draft_logits
            st[pre + "tokens"] = np.array(toks, dtype=np.int32)
            st[pre + "uniforms"] = uni
            st[pre + "path"] = np.array(res.accepted_path, dtype=np.int32)
            st[pre + "next"] = np.array(res.next_token)
            st[pre + "used"] = np.array(res.uniforms_used)
            st[pre + "residual"] = res.residual
            st[pre + "dist0"] = dists[0]
            k += 1
    st["n_cases"] = np.array(k)
    np.savez_compressed(os.path.join(OUT, "accept_stochastic.npz"), **st)

    # top-p / sample_from known answers on random dists (sampling.py:57-72, 105-109)
    rng2 = np.random.default_rng(9)
    d = rng2.dirichlet(np.ones(300) * 0.3, size=12)
    d[3] = 1.0 / 300  # all ties
    ps = np.array([0.1, 0.5, 0.9, 0.95, 0.999, 1.0, 0.3, 0.77, 0.6, 0.9, 0.01, 0.5])
    tp = np.stack([R_smp.top_p_mask(d[i], ps[i]) for i in range(12)])
    us = rng2.random(12)
    sf = np.array([R_smp.sample_from(d[i], us[i]) for i in range(12)])
    np.savez_compressed(os.path.join(OUT, "sampling_kat.npz"), dists=d, ps=ps, top_p=tp, us=us, sample=sf)


# ---------------------------------------------------------------------------
def gen_philox():
    specs = [(0, 0, 1, 5), (7, 3, 2, 5), (7, 3, 8, 5), (12345, 2, 4, 65), (2**40 + 3, 129, 3, 7),
             (2**63 - 1, 2**62, 2, 9)]
    out = {}
    for i, (seed, step, b, w) in enumerate(specs):
        out[f"p{i}_spec"] = np.array([seed, step, b, w], dtype=np.uint64)
        out[f"p{i}_u"] = R_smp.rank_sliced_uniforms(seed, step, b, w)
    out["n"] = np.array(len(specs))
    np.savez_compressed(os.path.join(OUT, "philox.npz"), **out)


# ---------------------------------------------------------------------------
def gen_compact():
    """Engine bookkeeping write-back replayed on the reference PagedKvCache
    (engine.py:504-523 -> kvstore.py:217-225, 248-258)."""
    rng = np.random.default_rng(77)
    out = {}
    k = 0
    for bs in (16, 4, 64):
        for spec, L in ((TREE64, 40), (N8, 17), ("chain:3", 16), ("full:2,2", 1), ("empty", 33)):
            tree = R_tree.EMPTY_TREE if spec == "empty" else R_tree.parse_tree(spec)
            aug = R_eng._augment(tree)
            hkv, d = 2, 8
            n_layers = 2
            nb = 64
            cache = R_kv.PagedKvCache(n_layers, hkv * d, n_blocks=nb, block_size=bs)
            cache.new_seq(0)
            C = L - 1
            committed = [rng.normal(size=(C, hkv * d)) for _ in range(2 * n_layers)]
            cache.ensure(0, max(C, 1))
            for li in range(n_layers):
                if C:
                    cache.write(0, li, 0, committed[2 * li], committed[2 * li + 1])
            cache.set_len(0, L)
            cache.alloc_for_step(0, tree.n_nodes)
            table_before = list(cache._seqs[0].table)
            # a random root-to-node path and a stop truncation sometimes
            path = []
            cur = -1
            while True:
                kids = tree.children(cur)
                if not kids or rng.random() < 0.25:
                    break
                cur = kids[int(rng.integers(len(kids)))]
                path.append(cur)
            kept = len(path) + 1
            if rng.random() < 0.3 and kept > 1:
                kept = int(rng.integers(1, kept + 1))  # stop-token truncation (engine.py:509-512)
            tree_kv = [(rng.normal(size=(aug.n_nodes, hkv * d)), rng.normal(size=(aug.n_nodes, hkv * d)))
                       for _ in range(n_layers)]
            write_path = path[:kept - 1]
            rows = [0] + [1 + a for a in write_path]
            for li in range(n_layers):
                kk, vv = tree_kv[li]
                cache.write(0, li, L - 1, kk[rows], vv[rows])
            new_len = L + kept
            cache.rewind(0, new_len - 1)
            cache.set_len(0, new_len)
            got = [cache.gather(0, li, new_len - 1) for li in range(n_layers)]
            pre = f"k{k}_"
            out[pre + "meta"] = np.array([bs, L, hkv, d, n_layers, nb, kept])
            out[pre + "parent"] = np.array(tree.parent, dtype=np.int32)
            out[pre + "path"] = np.array(path, dtype=np.int32)
            out[pre + "table"] = np.array(table_before, dtype=np.int32)
            out[pre + "table_after"] = np.array(cache._seqs[0].table, dtype=np.int32)
            for li in range(n_layers):
                out[pre + f"ck{li}"] = committed[2 * li]
                out[pre + f"cv{li}"] = committed[2 * li + 1]
                out[pre + f"tk{li}"] = tree_kv[li][0]
                out[pre + f"tv{li}"] = tree_kv[li][1]
                out[pre + f"gk{li}"] = got[li][0]
                out[pre + f"gv{li}"] = got[li][1]
            k += 1
    out["n_cases"] = np.array(k)
    np.savez_compressed(os.path.join(OUT, "compact.npz"), **out)


def gen_draft_attention():
    """Draft stage depth steps (engine.py:424-432 -> model.py:257-270): the
    new nodes of each depth attend the draft-cache prefix (CausalPrefix) and
    the carried ++ new suffix under the engine's vis-row mask (built here
    exactly like draft_stage, engine.py:409-421), merged with the
    reference's merge_attentions."""
    rng = np.random.default_rng(909)
    store = {}
    k = 0
    for spec, hq, hkv, d, ctx in ((TREE64, 8, 2, 16, 40), (N8, 4, 1, 8, 0), ("chain:4", 4, 2, 8, 17)):
        tree = R_tree.parse_tree(spec)
        parent = tree.parent
        n = len(parent)
        depth = [0] * n
        vis = []
        for i, p in enumerate(parent):
            depth[i] = 1 if p == R_tree.ROOT else depth[p] + 1
            row = np.zeros(i + 1, dtype=bool)
            if p != R_tree.ROOT:
                row[:p + 1] = vis[p]
            row[i] = True
            vis.append(row)
        g = hq // hkv

        def rep(x):
            return np.repeat(x.reshape(x.shape[0], hkv, d), g, axis=1).reshape(x.shape[0], hq * d)

        ck = bf16_round(rng.normal(size=(ctx, hkv * d)))
        cv = bf16_round(rng.normal(size=(ctx, hkv * d)))
        sk = bf16_round(rng.normal(size=(n, hkv * d)))
        sv = bf16_round(rng.normal(size=(n, hkv * d)))
        q = bf16_round(rng.normal(size=(n, hq * d)))
        scale = d ** -0.5
        for dep in range(1, max(depth) + 1):
            new = [i for i in range(n) if depth[i] == dep]
            total = new[-1] + 1
            mask = np.zeros((len(new), total), dtype=bool)
            for j, real in enumerate(new):
                mask[j, :real + 1] = vis[real]
            parts = []
            if ctx > 0:
                parts.append(R_att.attend(q[new], rep(ck), rep(cv), R_att.CausalPrefix(ctx), scale, hq))
            parts.append(R_att.attend(q[new], rep(sk[:total]), rep(sv[:total]), R_att.TreeSuffix(mask), scale, hq))
            m = R_att.merge_partials(parts, hq)  # merge_attentions == merge_partials(...).out
            pre = f"d{k}_"
            store.update({pre + "meta": np.array([hq, hkv, d, ctx, new[0], total]), pre + "parent": np.array(parent),
                          pre + "q": q[new], pre + "ck": ck, pre + "cv": cv, pre + "sk": sk[:total],
                          pre + "sv": sv[:total], pre + "mask": mask, pre + "out": m.out, pre + "lse": m.lse})
            k += 1
    store["n_cases"] = np.array(k)
    np.savez_compressed(os.path.join(OUT, "draft_attention.npz"), **store)


def gen_bookkeep():
    """Several engine rounds of bookkeeping on the reference caches
    (engine.py:455-457 alloc_for_step, 504-533 write-back / rewind / set_len
    for the base AND draft caches and the hidden tape, kvstore.py:195-258,
    389-431).  The draft cache's alignment write at L - 1 (draft_stage's
    first forward, engine.py:358-360) is replayed as a plain write."""
    rng = np.random.default_rng(4242)
    out = {}
    k = 0
    for bs, spec in ((16, TREE64), (4, N8), (8, "chain:3")):
        tree = R_tree.parse_tree(spec)
        aug = R_eng._augment(tree)
        hkv, d, n_layers, dim, nb = 2, 8, 2, 16, 96
        base = R_kv.PagedKvCache(n_layers, hkv * d, n_blocks=nb, block_size=bs)
        dr = R_kv.PagedKvCache(n_layers, hkv * d, n_blocks=nb, block_size=bs)
        tape = R_kv.HiddenTape(dim)
        for c in (base, dr):
            c.new_seq(0)
        L = 9  # committed length after prefill
        for c in (base, dr):
            c.ensure(0, L)
            for li in range(n_layers):
                c.write(0, li, 0, rng.normal(size=(L, hkv * d)), rng.normal(size=(L, hkv * d)))
            c.set_len(0, L)
        # prefill leaves L - 1 committed K/V rows: drop the last (it is the root of round 1)
        for c in (base, dr):
            c.rewind(0, L - 1)
            c.set_len(0, L)
        tape.append_rows(rng.normal(size=(L - 1, dim)))
        pre = f"b{k}_"
        out[pre + "meta"] = np.array([bs, hkv, d, n_layers, dim, nb, L])
        out[pre + "parent"] = np.array(tree.parent, dtype=np.int32)
        init_b = [base.gather(0, li, L - 1) for li in range(n_layers)]
        init_d = [dr.gather(0, li, L - 1) for li in range(n_layers)]
        for li in range(n_layers):
            out[pre + f"ib{li}"] = np.stack(init_b[li])
            out[pre + f"id{li}"] = np.stack(init_d[li])
        out[pre + "itape"] = tape.slice(0, len(tape))
        rounds = 4
        for rd in range(rounds):
            L = base.committed_len(0)
            base.alloc_for_step(0, tree.n_nodes)
            dr.alloc_for_step(0, tree.n_nodes)
            align = (rng.normal(size=(1, hkv * d)), rng.normal(size=(1, hkv * d)))
            for li in range(n_layers):
                dr.write(0, li, L - 1, align[0], align[1])
            path, cur = [], -1
            while True:
                kids = tree.children(cur)
                if not kids or rng.random() < 0.2:
                    break
                cur = kids[int(rng.integers(len(kids)))]
                path.append(cur)
            kept = len(path) + 1
            if rng.random() < 0.3 and kept > 1:
                kept = int(rng.integers(1, kept + 1))
            base_kv = [(rng.normal(size=(aug.n_nodes, hkv * d)), rng.normal(size=(aug.n_nodes, hkv * d)))
                       for _ in range(n_layers)]
            suf_kv = [(rng.normal(size=(tree.n_nodes, hkv * d)), rng.normal(size=(tree.n_nodes, hkv * d)))
                      for _ in range(n_layers)]
            hid = rng.normal(size=(aug.n_nodes, dim))
            write_path = path[:kept - 1]
            rows = [0] + [1 + a for a in write_path]
            for li in range(n_layers):
                base.write(0, li, L - 1, base_kv[li][0][rows], base_kv[li][1][rows])
            new_len = L + kept
            base.rewind(0, new_len - 1)
            base.set_len(0, new_len)
            if write_path:
                for li in range(n_layers):
                    dr.write(0, li, L, suf_kv[li][0][write_path], suf_kv[li][1][write_path])
            dr.rewind(0, new_len - 1)
            dr.set_len(0, new_len)
            tape.append_rows(np.stack([hid[0]] + [hid[1 + a] for a in write_path]))
            q = f"{pre}r{rd}_"
            out[q + "path"] = np.array(path, dtype=np.int32)
            out[q + "kept"] = np.array(kept)
            out[q + "align_k"], out[q + "align_v"] = align
            out[q + "hid"] = hid
            for li in range(n_layers):
                out[q + f"bk{li}"], out[q + f"bv{li}"] = base_kv[li]
                out[q + f"sk{li}"], out[q + f"sv{li}"] = suf_kv[li]
        L = base.committed_len(0)
        for li in range(n_layers):
            out[pre + f"gb{li}"] = np.stack(base.gather(0, li, L - 1))
            out[pre + f"gd{li}"] = np.stack(dr.gather(0, li, L - 1))
        out[pre + "tape"] = tape.slice(0, len(tape))
        out[pre + "final_len"] = np.array(L)
        out[pre + "blocks_used"] = np.array([len(base._seqs[0].table), len(dr._seqs[0].table)])
        out[pre + "rounds"] = np.array(rounds)
        k += 1
    out["n_cases"] = np.array(k)
    np.savez_compressed(os.path.join(OUT, "bookkeep.npz"), **out)


if __name__ == "__main__":
    os.makedirs(OUT, exist_ok=True)
    if len(sys.argv) > 1:  # e.g. `make_golden.py gen_draft_attention`
        for name in sys.argv[1:]:
            globals()[name]()
        sys.exit(0)
    gen_trees()
    gen_attention_f64()
    gen_attention_gqa()
    gen_accept()
    gen_philox()
    gen_compact()
    gen_draft_attention()
    gen_bookkeep()
    for f in sorted(os.listdir(OUT)):
        print(f, os.path.getsize(os.path.join(OUT, f)))
