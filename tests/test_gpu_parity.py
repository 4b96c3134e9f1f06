"""GPU parity: the CUDA path vs the reference's golden outputs and the CPU
oracle, through the package API (which calls the C ABI).  Needs a B200."""

import numpy as np
import pytest

torch = pytest.importorskip("torch")

pytestmark = pytest.mark.gpu

from oracle import specdec_oracle as O  # noqa: E402


@pytest.fixture(scope="module", autouse=True)
def _lib_loaded():
    from paper_2508_08192_b200 import _lib

    _lib.load()


def _cuda(x, dtype):
    return torch.as_tensor(np.ascontiguousarray(x)).to(device="cuda", dtype=dtype)


# ---------------------------------------------------------------------------
# K0 tree build
# ---------------------------------------------------------------------------

def test_tree_build_matches_reference(golden):
    from paper_2508_08192_b200.drafttree import tree_build

    g = golden("trees")
    par = _cuda(g["parent_aug"], torch.int32)
    nr = _cuda(g["n_rows"], torch.int32)
    ctx = _cuda(g["ctx"], torch.int32)
    mask, pos, depth, err = tree_build(par, nr, ctx)
    torch.cuda.synchronize()
    assert int(err.abs().sum()) == 0
    mask, pos, depth = mask.cpu().numpy(), pos.cpu().numpy(), depth.cpu().numpy()
    for i in range(len(g["n_rows"])):
        n = int(g["n_rows"][i])
        want = O.mask_words(g["mask"][i, :n, :n], mask.shape[-1])
        np.testing.assert_array_equal(mask[i, :n].astype(np.uint32), want)
        np.testing.assert_array_equal(depth[i, :n], g["depth"][i, :n])
        np.testing.assert_array_equal(pos[i, :n], g["pos"][i, :n])
        assert not mask[i, n:].any()


def test_tree_build_rejects_bad_parents(golden):
    from paper_2508_08192_b200.drafttree import tree_build

    g = golden("trees")
    mask, pos, depth, err = tree_build(_cuda(g["bad_parent"], torch.int32), _cuda(g["bad_len"], torch.int32))
    err = err.cpu().numpy()
    np.testing.assert_array_equal(err == 0, g["bad_valid"])


def test_suffix_mask_drop_in_known_answers():
    from paper_2508_08192_b200 import drafttree as D

    t = D.augment(D.parse_tree("full:2,2"))
    m = D.suffix_mask(t)
    assert list(O.mask_words(m)[:, 0]) == [1, 3, 5, 11, 19, 37, 69]
    with pytest.raises(D.TreeError):
        D.TreeSpec((-1, 2, 1))
    # reference tests/test_drafttree.py:53-61
    t = D.parse_tree("full:2,2")
    m = D.suffix_mask(t)
    for i in range(t.n_nodes):
        expect = np.zeros(t.n_nodes, dtype=bool)
        expect[t.ancestors_or_self(i)] = True
        np.testing.assert_array_equal(m[i], expect)
    assert not np.triu(m, 1).any()


# ---------------------------------------------------------------------------
# drop-in float64 attention (reference tolerances)
# ---------------------------------------------------------------------------

def _softmax_ref(q, k, v, mask, scale):
    s = (q @ k.T) * scale
    if mask is not None:
        s = np.where(mask, s, -np.inf)
    s = s - s.max(axis=1, keepdims=True)
    p = np.exp(s)
    p /= p.sum(axis=1, keepdims=True)
    return p @ v


def test_attend_reference_cases():
    from paper_2508_08192_b200.attention import (AttentionError, CausalPrefix, LocalChunk, TreeSuffix, attend,
                                                 merge_attentions, merge_partials)

    # tests/test_attention.py:22-85 of the reference, same tolerances
    rng = np.random.default_rng(0)
    q, k, v = (rng.normal(size=(3, 8)) for _ in range(3))
    np.testing.assert_allclose(attend(q, k, v, CausalPrefix(3), 0.5).out, _softmax_ref(q, k, v, None, 0.5),
                               atol=1e-12)
    rng = np.random.default_rng(1)
    q1 = rng.normal(size=(1, 4))
    k1, v1 = rng.normal(size=(6, 4)), rng.normal(size=(6, 4))
    mask = np.zeros((1, 6), dtype=bool)
    mask[0, 4:6] = True
    np.testing.assert_allclose(attend(q1, k1, v1, LocalChunk(4, (5,), tuple(range(6))), 1.0).out,
                               _softmax_ref(q1, k1, v1, mask, 1.0), atol=1e-12)
    part = attend(np.ones((2, 4)), np.zeros((0, 4)), np.zeros((0, 4)), CausalPrefix(0), 1.0)
    assert part.masked_rows.all()
    rng = np.random.default_rng(2)
    q = rng.normal(size=(4, 8))
    k, v = rng.normal(size=(10, 8)), rng.normal(size=(10, 8))
    for cut in (1, 3, 7, 9):
        a = attend(q, k[:cut], v[:cut], CausalPrefix(cut), 0.3)
        b = attend(q, k[cut:], v[cut:], CausalPrefix(10 - cut), 0.3)
        np.testing.assert_allclose(merge_attentions([a, b]), attend(q, k, v, CausalPrefix(10), 0.3).out, atol=1e-10)
    rng = np.random.default_rng(3)
    q = rng.normal(size=(2, 8))
    k, v = rng.normal(size=(6, 8)), rng.normal(size=(6, 8))
    a = attend(q, k[:2], v[:2], CausalPrefix(2), 1.0, n_heads=2)
    b = attend(q, k[2:], v[2:], CausalPrefix(4), 1.0, n_heads=2)
    np.testing.assert_allclose(merge_attentions([a, b], n_heads=2),
                               attend(q, k, v, CausalPrefix(6), 1.0, n_heads=2).out, atol=1e-10)
    empty = attend(np.ones((1, 4)), np.zeros((0, 4)), np.zeros((0, 4)), CausalPrefix(0), 1.0)
    with pytest.raises(AttentionError):
        merge_partials([empty, empty])
    with pytest.raises(AttentionError):
        attend(np.ones((2, 4)), np.ones((3, 4)), np.ones((3, 4)), TreeSuffix(np.ones((2, 2), dtype=bool)), 1.0)


def test_attend_merge_golden(golden):
    from paper_2508_08192_b200.attention import CausalPrefix, TreeSuffix, attend, merge_partials

    g = golden("attend_merge")
    q, k, v = g["q"], g["k"], g["v"]
    a = attend(q, k[:3], v[:3], CausalPrefix(3), 0.3, n_heads=2)
    b = attend(q, k[3:], v[3:], CausalPrefix(7), 0.3, n_heads=2)
    np.testing.assert_allclose(a.out, g["a_out"], atol=1e-13)
    np.testing.assert_allclose(b.lse, g["b_lse"], atol=1e-13)
    m = merge_partials([a, b], n_heads=2)
    np.testing.assert_allclose(m.out, g["m_out"], atol=1e-13)
    np.testing.assert_allclose(m.lse, g["m_lse"], atol=1e-13)
    c = attend(q, k, v, TreeSuffix(g["mask"]), 0.3, n_heads=2)
    np.testing.assert_allclose(c.out, g["c_out"], atol=1e-13)
    np.testing.assert_array_equal(np.isinf(c.lse), np.isinf(g["c_lse"]))


def test_tree_attention_f64_golden(golden):
    from paper_2508_08192_b200.attention import tree_attention
    from paper_2508_08192_b200.drafttree import TreeSpec

    g = golden("attention_f64")
    for ci in range(int(g["n_cases"])):
        p = f"c{ci}_"
        nh, hd, ctx, chunk = (int(x) for x in g[p + "meta"])
        tree = TreeSpec(tuple(int(x) for x in g[p + "parent"]))
        out = tree_attention(g[p + "q"], g[p + "ck"], g[p + "cv"], g[p + "tk"], g[p + "tv"], tree, hd ** -0.5,
                             n_heads=nh, chunk_len=None if chunk < 0 else chunk)
        # reference suite threshold is 1e-5 (verify.py:284); float64 gives far better
        np.testing.assert_allclose(out, g[p + "out"], atol=1e-12, rtol=0)


def test_tree_attention_vs_naive_randomized():
    # reference tests/test_attention.py:88-111 through the device path
    from paper_2508_08192_b200.attention import explicit_tree_mask, naive_tree_attention, tree_attention
    from paper_2508_08192_b200.drafttree import ROOT, TreeSpec

    rng = np.random.default_rng(5)
    for case in range(20):
        n_nodes = int(rng.integers(1, 17))
        parent = [ROOT]
        for i in range(1, n_nodes):
            parent.append(int(rng.integers(0, i)) if rng.random() < 0.8 else ROOT)
        tree = TreeSpec(tuple(parent))
        ctx = int(rng.integers(0, 65))
        heads = int(rng.choice([1, 2, 4]))
        dh = int(rng.choice([4, 8]))
        dim = heads * dh
        chunk = None if case % 2 == 0 else int(rng.choice([4, 8]))
        q = rng.normal(size=(n_nodes, dim))
        ck, cv = rng.normal(size=(ctx, dim)), rng.normal(size=(ctx, dim))
        tk, tv = rng.normal(size=(n_nodes, dim)), rng.normal(size=(n_nodes, dim))
        got = tree_attention(q, ck, cv, tk, tv, tree, dh ** -0.5, n_heads=heads, chunk_len=chunk)
        mask = explicit_tree_mask(tree, ctx, chunk_len=chunk)
        want = naive_tree_attention(q, np.concatenate([ck, tk]), np.concatenate([cv, tv]), mask, dh ** -0.5,
                                    n_heads=heads)
        assert np.max(np.abs(got - want)) < 1e-5


# ---------------------------------------------------------------------------
# batched paged GQA tree-verify attention
# ---------------------------------------------------------------------------

def _gqa_case(g, name, dtype):
    from paper_2508_08192_b200.drafttree import tree_build

    p = name + "_"
    bsz, hq, hkv, d, bs, r_max = (int(x) for x in g[p + "meta"])
    q = _cuda(g[p + "q"], dtype)
    kp = _cuda(g[p + "k_pool"], dtype)
    vp = _cuda(g[p + "v_pool"], dtype)
    tk = _cuda(g[p + "tk"], dtype)
    tv = _cuda(g[p + "tv"], dtype)
    table = _cuda(g[p + "table"], torch.int32)
    ctx = _cuda(g[p + "ctx"], torch.int32)
    par = _cuda(g[p + "parent_aug"], torch.int32)
    nr = _cuda(g[p + "n_rows"], torch.int32)
    mask, _pos, _depth, err = tree_build(par, nr, ctx)
    return dict(q=q, kp=kp, vp=vp, tk=tk, tv=tv, table=table, ctx=ctx, mask=mask, nr=nr, d=d,
                out=g[p + "out"], lse=g[p + "lse"], n_rows=g[p + "n_rows"])


@pytest.mark.parametrize("kernel", [0, 1, 2])
@pytest.mark.parametrize("splits", [0, 1, 3])
def test_tree_verify_attention_bf16_golden(golden, kernel, splits):
    """kernel 1 = tcgen05 (d = 128 cases), 2 = SIMT, 0 = auto."""
    from paper_2508_08192_b200.attention import tree_verify_attention

    g = golden("attention_gqa")
    for name in g["names"]:
        c = _gqa_case(g, str(name), torch.bfloat16)
        if kernel == 1 and c["d"] != 128:
            continue
        out, lse = tree_verify_attention(c["q"], c["kp"], c["vp"], c["table"], c["ctx"], c["tk"], c["tv"], c["mask"],
                                         c["nr"], c["d"] ** -0.5, num_splits=splits, kernel=kernel)
        torch.cuda.synchronize()
        out = out.float().cpu().numpy()
        lse = lse.cpu().numpy()
        for b, n in enumerate(c["n_rows"]):
            # bf16 output rounding: |x| <~ 3 -> 2^-7 relative
            np.testing.assert_allclose(out[b, :n], c["out"][b, :n], atol=2e-2, rtol=0)
            assert np.abs(out[b, :n] - c["out"][b, :n]).mean() < 2e-3
            np.testing.assert_allclose(lse[b, :, :n], c["lse"][b, :, :n], atol=1e-3, rtol=0)
            assert not out[b, n:].any()


@pytest.mark.parametrize("splits", [1, 4])
def test_tree_verify_attention_fp32_golden(golden, splits):
    from paper_2508_08192_b200.attention import tree_verify_attention

    g = golden("attention_gqa")
    for name in g["names"]:
        c = _gqa_case(g, str(name), torch.float32)
        out, lse = tree_verify_attention(c["q"], c["kp"], c["vp"], c["table"], c["ctx"], c["tk"], c["tv"], c["mask"],
                                         c["nr"], c["d"] ** -0.5, num_splits=splits, kernel=2)
        torch.cuda.synchronize()
        out, lse = out.cpu().numpy(), lse.cpu().numpy()
        for b, n in enumerate(c["n_rows"]):
            np.testing.assert_allclose(out[b, :n], c["out"][b, :n], atol=1e-5, rtol=0)
            np.testing.assert_allclose(lse[b, :, :n], c["lse"][b, :, :n], atol=1e-5, rtol=0)


# ---------------------------------------------------------------------------
# acceptance
# ---------------------------------------------------------------------------

def _aug_batch(parents, tokens_list, r_max):
    b = len(parents)
    par = np.full((b, r_max), -1, dtype=np.int32)
    tok = np.zeros((b, r_max), dtype=np.int32)
    nr = np.zeros((b,), dtype=np.int32)
    for i, (p, t) in enumerate(zip(parents, tokens_list)):
        aug = O.augment(tuple(int(x) for x in p))
        par[i, :len(aug)] = aug
        tok[i, 1:len(aug)] = t
        nr[i] = len(aug)
    return par, tok, nr


def test_accept_greedy_golden(golden):
    from paper_2508_08192_b200.sampling import accept_greedy

    g = golden("accept_greedy")
    for k in range(int(g["n_cases"])):
        p = f"g{k}_"
        logits = g[p + "logits"]
        n = logits.shape[0]
        par, tok, nr = _aug_batch([g[p + "parent"]], [g[p + "tokens"]], n)
        for dt in (torch.float32, torch.bfloat16):
            lg = _cuda(logits[None], dt)
            res = accept_greedy(lg, _cuda(par, torch.int32), _cuda(nr, torch.int32), _cuda(tok, torch.int32))
            plen = int(res.path_len[0])
            if dt == torch.float32:
                assert list(res.path[0, :plen].cpu().numpy()) == list(g[p + "path"])
                assert int(res.next_token[0]) == int(g[p + "next"])
                assert int(res.uniforms_used[0]) == int(g[p + "used"])
            else:
                # bf16 logits: compare with the oracle on the rounded logits
                am = np.argmax(lg[0].float().cpu().numpy().astype(np.float64), axis=1)
                path, nxt, used = O.greedy_walk(tuple(int(x) for x in g[p + "parent"]), g[p + "tokens"], am)
                assert list(res.path[0, :plen].cpu().numpy()) == path
                assert int(res.next_token[0]) == nxt and int(res.uniforms_used[0]) == used
            assert int(res.err[0]) == 0


def test_accept_greedy_batched_ragged(golden):
    """All golden cases in ONE batched launch (ragged R per sequence)."""
    from paper_2508_08192_b200.sampling import accept_greedy

    g = golden("accept_greedy")
    cases = [k for k in range(int(g["n_cases"])) if g[f"g{k}_logits"].shape[1] == 4096]
    r_max = max(g[f"g{k}_logits"].shape[0] for k in cases)
    lg = np.zeros((len(cases), r_max, 4096), dtype=np.float32)
    for i, k in enumerate(cases):
        lg[i, :g[f"g{k}_logits"].shape[0]] = g[f"g{k}_logits"]
    par, tok, nr = _aug_batch([g[f"g{k}_parent"] for k in cases], [g[f"g{k}_tokens"] for k in cases], r_max)
    res = accept_greedy(_cuda(lg, torch.float32), _cuda(par, torch.int32), _cuda(nr, torch.int32),
                        _cuda(tok, torch.int32))
    for i, k in enumerate(cases):
        plen = int(res.path_len[i])
        assert list(res.path[i, :plen].cpu().numpy()) == list(g[f"g{k}_path"])
        assert int(res.next_token[i]) == int(g[f"g{k}_next"])
        assert int(res.uniforms_used[i]) == int(g[f"g{k}_used"])


def test_accept_greedy_nan_raises_flag():
    from paper_2508_08192_b200.sampling import accept_greedy

    lg = torch.zeros((1, 2, 64), dtype=torch.float32, device="cuda")
    lg[0, 1, 5] = float("nan")
    par = torch.tensor([[-1, 0]], dtype=torch.int32, device="cuda")
    res = accept_greedy(lg, par, torch.tensor([2], dtype=torch.int32, device="cuda"),
                        torch.zeros((1, 2), dtype=torch.int32, device="cuda"))
    assert int(res.err[0]) & 2


def _margin_ok(g, k, res_path, res_next, res_used):
    return (list(res_path) == list(g[f"s{k}_path"]) and res_next == int(g[f"s{k}_next"])
            and res_used == int(g[f"s{k}_used"]))


@pytest.mark.parametrize("lazy", [True, False])
def test_accept_stochastic_golden(golden, lazy):
    """Stochastic acceptance vs the reference (fp32 pipeline; decisions whose
    reference margin is < 1e-6 may differ and are counted -- none expected
    on these fixtures); lazy (visited rows only) and eager (every row)."""
    from paper_2508_08192_b200.sampling import StochasticAcceptor

    def accept_stochastic(*a, **k):
        return StochasticAcceptor(lazy=lazy)(*a, **k)

    g = golden("accept_stochastic")
    mism = []
    for k in range(int(g["n_cases"])):
        p = f"s{k}_"
        temp, top_p, _seed = g[p + "meta"]
        logits, dl = g[p + "logits"], g[p + "draft_logits"]
        n = logits.shape[0]
        par, tok, nr = _aug_batch([g[p + "parent"]], [g[p + "tokens"]], n)
        res = accept_stochastic(_cuda(logits[None], torch.float32), _cuda(dl[None], torch.float32), float(temp),
                                float(top_p), _cuda(par, torch.int32), _cuda(nr, torch.int32),
                                _cuda(tok, torch.int32), _cuda(g[p + "uniforms"][None], torch.float64),
                                want_residual=True)
        torch.cuda.synchronize()
        assert int(res.err[0]) == 0
        plen = int(res.path_len[0])
        got = (res.path[0, :plen].cpu().numpy(), int(res.next_token[0]), int(res.uniforms_used[0]))
        if not _margin_ok(g, k, *got):
            mism.append((k, got, list(g[p + "path"]), int(g[p + "next"])))
        else:
            np.testing.assert_allclose(res.residual[0].cpu().numpy(), g[p + "residual"], atol=2e-6)
    assert not mism, mism


def test_target_dist_and_mss_drop_in(golden):
    from paper_2508_08192_b200 import sampling as S
    from paper_2508_08192_b200.drafttree import TreeSpec

    g = golden("sampling_kat")
    for i in range(len(g["ps"])):
        np.testing.assert_allclose(S.top_p_mask(g["dists"][i], g["ps"][i]), g["top_p"][i], atol=1e-12)
        assert S.sample_from(g["dists"][i], g["us"][i]) == int(g["sample"][i])
    # reference tests/test_sampling.py:11-58
    d = np.array([0.5, 0.3, 0.2])
    np.testing.assert_allclose(S.top_p_mask(d, 0.8), [0.625, 0.375, 0.0])
    np.testing.assert_allclose(S.top_p_mask(d, 0.5), [1.0, 0.0, 0.0])
    np.testing.assert_allclose(S.top_p_mask(d, 0.51), [0.625, 0.375, 0.0])
    np.testing.assert_allclose(S.top_p_mask(np.full(4, 0.25), 0.5), [0.5, 0.5, 0.0, 0.0])
    np.testing.assert_array_equal(S.target_dist(np.array([0.1, 3.0, -1.0]), 0.0, 1.0), [0, 1, 0])
    np.testing.assert_array_equal(S.target_dist(np.array([5.0, 1.0, 0.0]), 0.0, 1.0,
                                                np.array([False, True, True])), [0, 1, 0])
    with pytest.raises(S.SamplingError):
        S.target_dist(np.array([5.0, 1.0, 0.0]), 1.0, 1.0, np.zeros(3, dtype=bool))
    d = np.array([0.2, 0.5, 0.3])
    assert [S.sample_from(d, u) for u in (0.0, 0.19, 0.2, 0.69, 0.7, 0.999999)] == [0, 0, 1, 1, 2, 2]
    # MSS known answers (reference tests/test_sampling.py:79-138)
    q = np.array([0.5, 0.5, 0.0])
    p = np.array([0.6, 0.4, 0.0])
    chain2 = TreeSpec((-1, 0))
    r = S.mss_verify(S.DraftResult(chain2, (0, 0), (q, q)), [p, p, np.array([0.0, 0.0, 1.0])], [0.9, 0.9, 0.5])
    assert r.accepted_path == [0, 1] and r.next_token == 2 and r.uniforms_used == 3
    c1 = TreeSpec((-1,))
    r = S.mss_verify(S.DraftResult(c1, (0,), (np.array([1.0, 0.0]),)), [np.array([0.3, 0.7])] * 2, [0.5, 0.0])
    assert r.accepted_path == [] and r.next_token == 1
    np.testing.assert_allclose(r.residual, [0.0, 1.0])
    q1 = np.array([1.0, 0.0, 0.0])
    r = S.mss_verify(S.DraftResult(TreeSpec((-1, -1)), (0, 1), (q1, q1)), [np.array([0.0, 1.0, 0.0])] * 3,
                     [0.5] * 3)
    assert r.accepted_path == [1] and r.next_token == 1
    r = S.mss_verify(S.DraftResult(c1, (0,), (np.array([1.0, 0.0]),)), [np.array([1.0, 0.0])] * 2, [1.0, 0.3])
    assert r.accepted_path == [] and r.next_token == 0
    with pytest.raises(S.SamplingError):
        S.mss_verify(S.DraftResult(c1, (0,), (np.array([0.5, 0.5]),)), [np.array([0.5, 0.5])] * 2, [0.5])


def test_mss_drop_in_matches_reference_golden(golden):
    from paper_2508_08192_b200 import sampling as S
    from paper_2508_08192_b200.drafttree import TreeSpec

    g = golden("accept_stochastic")
    for k in range(int(g["n_cases"])):
        p = f"s{k}_"
        temp, top_p, _seed = g[p + "meta"]
        parent = tuple(int(x) for x in g[p + "parent"])
        logits, dl = g[p + "logits"], g[p + "draft_logits"]
        qd = [S.target_dist(dl[0 if a == -1 else 1 + a], temp, 1.0) for a in parent]
        dists = list(S.target_dists(logits, temp, top_p))
        np.testing.assert_allclose(dists[0], g[p + "dist0"], atol=1e-14)
        r = S.mss_verify(S.DraftResult(TreeSpec(parent), tuple(g[p + "tokens"]), tuple(qd)), dists, g[p + "uniforms"],
                         mode="stochastic")
        assert r.accepted_path == list(g[p + "path"])
        assert r.next_token == int(g[p + "next"]) and r.uniforms_used == int(g[p + "used"])
        np.testing.assert_allclose(r.residual, g[p + "residual"], atol=1e-12)


# ---------------------------------------------------------------------------
# K7 compaction + paged cache
# ---------------------------------------------------------------------------

def test_paged_cache_and_compaction_golden(golden):
    from paper_2508_08192_b200.kvstore import PagedKvCache, compact_kv

    g = golden("compact")
    for k in range(int(g["n_cases"])):
        p = f"k{k}_"
        bs, L, hkv, d, n_layers, nb, kept = (int(x) for x in g[p + "meta"])
        table = g[p + "table"]
        path = [int(x) for x in g[p + "path"]]
        C = L - 1
        # drop-in cache replaying the engine's write-back
        cache = PagedKvCache(n_layers, hkv * d, n_blocks=nb, block_size=bs)
        cache.new_seq(0)
        cache.ensure(0, max(C, 1))
        for li in range(n_layers):
            if C:
                cache.write(0, li, 0, g[p + f"ck{li}"], g[p + f"cv{li}"])
        cache.set_len(0, L)
        n_tree = g[p + f"tk0"].shape[0]
        cache.alloc_for_step(0, n_tree - 1)
        assert cache.block_table(0) == list(table)
        rows = O.accepted_rows(path, kept)
        for li in range(n_layers):
            cache.write(0, li, L - 1, g[p + f"tk{li}"][rows], g[p + f"tv{li}"][rows])
        cache.rewind(0, L + kept - 1)
        cache.set_len(0, L + kept)
        assert cache.block_table(0) == list(g[p + "table_after"])
        for li in range(n_layers):
            gk, gv = cache.gather(0, li, L + kept - 1)
            np.testing.assert_array_equal(gk, g[p + f"gk{li}"])
            np.testing.assert_array_equal(gv, g[p + f"gv{li}"])
        # batched device compaction on the head-split layout (bf16-exact data)
        kpool = torch.zeros((n_layers, nb, hkv, bs, d), dtype=torch.float32, device="cuda")
        vpool = torch.zeros_like(kpool)
        tk = torch.zeros((n_layers, 1, n_tree, hkv, d), dtype=torch.float32, device="cuda")
        tv = torch.zeros_like(tk)
        want_k = np.zeros((n_layers, nb, hkv, bs, d))
        want_v = np.zeros_like(want_k)
        for li in range(n_layers):
            tk[li, 0] = _cuda(g[p + f"tk{li}"].reshape(n_tree, hkv, d), torch.float32)
            tv[li, 0] = _cuda(g[p + f"tv{li}"].reshape(n_tree, hkv, d), torch.float32)
            O.compact_kv(want_k[li], want_v[li], table, C, g[p + f"tk{li}"].reshape(n_tree, hkv, d).astype(np.float32),
                         g[p + f"tv{li}"].reshape(n_tree, hkv, d).astype(np.float32), path, kept)
        pt = np.zeros((1, n_tree), dtype=np.int32)
        pt[0, :len(path)] = path
        compact_kv(tk, tv, kpool, vpool, _cuda(table[None], torch.int32), _cuda([C], torch.int32),
                   _cuda(pt, torch.int32), _cuda([len(path)], torch.int32), _cuda([kept], torch.int32))
        np.testing.assert_array_equal(kpool.cpu().numpy(), want_k.astype(np.float32))
        np.testing.assert_array_equal(vpool.cpu().numpy(), want_v.astype(np.float32))


def _rand_paged_case(B, Hq, Hkv, d, C_max, bs, parent_raw, seed, ragged=True):
    from paper_2508_08192_b200.drafttree import tree_build

    rng = np.random.default_rng(seed)
    aug = O.augment(tuple(parent_raw))
    R = len(aug)
    ctx = (rng.integers(C_max // 2, C_max + 1, size=B) if ragged else np.full(B, C_max)).astype(np.int32)
    pages = -(-(C_max + R) // bs)
    nb = B * pages + 5
    table = rng.permutation(nb)[:B * pages].reshape(B, pages).astype(np.int32)
    gen = torch.Generator(device="cuda").manual_seed(seed)
    kp = torch.randn((nb, Hkv, bs, d), generator=gen, device="cuda").to(torch.bfloat16)
    vp = torch.randn((nb, Hkv, bs, d), generator=gen, device="cuda").to(torch.bfloat16)
    q = torch.randn((B, R, Hq, d), generator=gen, device="cuda").to(torch.bfloat16)
    tk = torch.randn((B, R, Hkv, d), generator=gen, device="cuda").to(torch.bfloat16)
    tv = torch.randn((B, R, Hkv, d), generator=gen, device="cuda").to(torch.bfloat16)
    par = torch.tensor([list(aug)] * B, dtype=torch.int32, device="cuda")
    nr = torch.full((B,), R, dtype=torch.int32, device="cuda")
    ctx_t = torch.tensor(ctx, device="cuda")
    mask, _, _, _ = tree_build(par, nr, ctx_t)
    return dict(q=q, kp=kp, vp=vp, tk=tk, tv=tv, table=torch.tensor(table, device="cuda"), ctx=ctx_t, mask=mask,
                nr=nr, aug=aug, ctx_np=ctx, table_np=table, R=R)


TREE64 = [-1, -1, -1, -1, -1, -1, -1, -1, 0, 0, 0, 0, 0, 0, 1, 1, 1, 1, 1, 2, 2, 2, 2, 3, 3, 3, 4, 4, 5, 5, 6, 7,
          8, 8, 8, 8, 9, 9, 9, 10, 10, 10, 11, 11, 12, 13, 14, 15, 32, 32, 32, 33, 33, 34, 34, 35, 36, 37, 48, 48, 49,
          50, 51]


@pytest.mark.parametrize("bs,splits", [(64, 1), (16, 3), (128, 0)])
def test_tcgen05_llama70b_shapes_vs_oracle(bs, splits):
    """70B attention shapes (64q/8kv, d128, 64-row tree) at 8k ragged context
    through the tcgen05 kernel vs the float64 oracle (bf16 tolerance)."""
    from paper_2508_08192_b200.attention import tree_verify_attention

    c = _rand_paged_case(2, 64, 8, 128, 8192, bs, TREE64, seed=11)
    out, lse = tree_verify_attention(c["q"], c["kp"], c["vp"], c["table"], c["ctx"], c["tk"], c["tv"], c["mask"],
                                     c["nr"], 128 ** -0.5, num_splits=splits, kernel=1)
    torch.cuda.synchronize()
    f64 = lambda t: t.float().cpu().numpy().astype(np.float64)
    want_o, want_l = O.tree_verify_attention_batch(f64(c["q"]), f64(c["kp"]), f64(c["vp"]), c["table_np"],
                                                   c["ctx_np"], f64(c["tk"]), f64(c["tv"]), [c["aug"]] * 2,
                                                   128 ** -0.5)
    got_o = out.float().cpu().numpy()
    err = np.abs(got_o - want_o)
    assert err.max() < 2e-2 and err.mean() < 2e-3, (err.max(), err.mean())
    assert np.abs(lse.cpu().numpy() - want_l).max() < 2e-3


def test_tcgen05_matches_simt_on_device():
    """Same inputs through both device kernels (larger batch, chain and N8 trees)."""
    from paper_2508_08192_b200.attention import tree_verify_attention

    for tree, hq, hkv in (([-1, 0, 1], 64, 8), ([-1, -1, 0, 0, 1, 2, 2, 5], 32, 8), (TREE64, 16, 16)):
        c = _rand_paged_case(5, hq, hkv, 128, 3000, 32, tree, seed=len(tree))
        o1, l1 = tree_verify_attention(c["q"], c["kp"], c["vp"], c["table"], c["ctx"], c["tk"], c["tv"], c["mask"],
                                       c["nr"], 0.088, kernel=1)
        o2, l2 = tree_verify_attention(c["q"], c["kp"], c["vp"], c["table"], c["ctx"], c["tk"], c["tv"], c["mask"],
                                       c["nr"], 0.088, kernel=2)
        torch.cuda.synchronize()
        assert (o1.float() - o2.float()).abs().max().item() < 2e-2
        assert (l1 - l2).abs().max().item() < 2e-3


@pytest.mark.parametrize("ctas", [0, 7, 148])
def test_tcgen05_small_batch_stream_k(ctas):
    """bs1 (8B shapes, 32q/8kv): each unit spans many persistent CTAs, so the
    fix-up merges long chains of partial pieces."""
    from paper_2508_08192_b200.attention import tree_verify_attention

    c = _rand_paged_case(1, 32, 8, 128, 4096, 64, TREE64, seed=3, ragged=False)
    out, lse = tree_verify_attention(c["q"], c["kp"], c["vp"], c["table"], c["ctx"], c["tk"], c["tv"], c["mask"],
                                     c["nr"], 128 ** -0.5, num_splits=ctas, kernel=1)
    torch.cuda.synchronize()
    f64 = lambda t: t.float().cpu().numpy().astype(np.float64)
    want_o, want_l = O.tree_verify_attention_batch(f64(c["q"]), f64(c["kp"]), f64(c["vp"]), c["table_np"],
                                                   c["ctx_np"], f64(c["tk"]), f64(c["tv"]), [c["aug"]], 128 ** -0.5)
    err = np.abs(out.float().cpu().numpy() - want_o)
    assert err.max() < 2e-2 and err.mean() < 2e-3, (err.max(), err.mean())
    assert np.abs(lse.cpu().numpy() - want_l).max() < 2e-3


def test_tcgen05_fixup_more_split_units_than_listed():
    """250 CTA-pair workers over 256 units (B 16, 64q/8kv: two 256-row blocks
    per KV head): ~250 split units, more than the host list holds, so the
    fix-up falls back to one block row per worker boundary."""
    from paper_2508_08192_b200.attention import tree_verify_attention

    c = _rand_paged_case(16, 64, 8, 128, 512, 64, TREE64, seed=5, ragged=True)
    out, lse = tree_verify_attention(c["q"], c["kp"], c["vp"], c["table"], c["ctx"], c["tk"], c["tv"], c["mask"],
                                     c["nr"], 128 ** -0.5, num_splits=250, kernel=1)
    torch.cuda.synchronize()
    f64 = lambda t: t.float().cpu().numpy().astype(np.float64)
    want_o, want_l = O.tree_verify_attention_batch(f64(c["q"]), f64(c["kp"]), f64(c["vp"]), c["table_np"],
                                                   c["ctx_np"], f64(c["tk"]), f64(c["tv"]), [c["aug"]] * 16,
                                                   128 ** -0.5)
    err = np.abs(out.float().cpu().numpy() - want_o)
    assert err.max() < 2e-2 and err.mean() < 2e-3, (err.max(), err.mean())
    assert np.abs(lse.cpu().numpy() - want_l).max() < 2e-3


@pytest.mark.parametrize("group", ["1", "2"])
def test_tcgen05_single_cta_and_pair_kernels_agree(group, monkeypatch):
    """Force the 1-CTA (M=128) or the CTA-pair (cta_group::2, M=256) kernel on
    the same 70B-shaped inputs; both must match the float64 oracle."""
    from paper_2508_08192_b200.attention import tree_verify_attention

    monkeypatch.setenv("SDB_ATTN_CTA_GROUP", group)
    c = _rand_paged_case(3, 64, 8, 128, 2048, 32, TREE64, seed=21)
    out, lse = tree_verify_attention(c["q"], c["kp"], c["vp"], c["table"], c["ctx"], c["tk"], c["tv"], c["mask"],
                                     c["nr"], 128 ** -0.5, kernel=1)
    torch.cuda.synchronize()
    f64 = lambda t: t.float().cpu().numpy().astype(np.float64)
    want_o, want_l = O.tree_verify_attention_batch(f64(c["q"]), f64(c["kp"]), f64(c["vp"]), c["table_np"],
                                                   c["ctx_np"], f64(c["tk"]), f64(c["tv"]), [c["aug"]] * 3,
                                                   128 ** -0.5)
    err = np.abs(out.float().cpu().numpy() - want_o)
    assert err.max() < 2e-2 and err.mean() < 2e-3, (err.max(), err.mean())
    assert np.abs(lse.cpu().numpy() - want_l).max() < 2e-3


# ---------------------------------------------------------------------------
# Draft-side tree attention: the draft stage's depth step
# -- new nodes attend prefix + carried/new suffix under a rectangular mask
# ---------------------------------------------------------------------------

def _depths(parent):
    d = []
    for p in parent:
        d.append(1 if p < 0 else d[p] + 1)
    return d


@pytest.mark.parametrize("kernel,dtype,hq,hkv,d", [(1, torch.bfloat16, 64, 8, 128), (2, torch.bfloat16, 32, 8, 128),
                                                    (2, torch.float32, 8, 2, 64)])
def test_draft_depth_attention_vs_oracle(kernel, dtype, hq, hkv, d):
    """Every depth of a realized draft tree (the 63-node EAGLE shape without
    the root, plus a ragged chain) as one rectangular call per depth:
    rows [q0, total) vs the float64 oracle of model.py:257-270; rows < q0
    are left untouched."""
    from paper_2508_08192_b200.attention import draft_tree_attention
    from paper_2508_08192_b200.drafttree import tree_build

    trees = [tuple(TREE64), (-1, 0, 1, 2, 3)]
    B, bs = len(trees), 32
    R = max(len(t) for t in trees)
    rng = np.random.default_rng(7)
    ctx = np.array([1500, 777], dtype=np.int32)
    pages = -(-(int(ctx.max()) + 1) // bs)
    nb = B * pages + 3
    table = rng.permutation(nb)[:B * pages].reshape(B, pages).astype(np.int32)
    gen = torch.Generator(device="cuda").manual_seed(5)
    kp = torch.randn((nb, hkv, bs, d), generator=gen, device="cuda").to(dtype)
    vp = torch.randn((nb, hkv, bs, d), generator=gen, device="cuda").to(dtype)
    q = torch.randn((B, R, hq, d), generator=gen, device="cuda").to(dtype)
    sk = torch.randn((B, R, hkv, d), generator=gen, device="cuda").to(dtype)
    sv = torch.randn((B, R, hkv, d), generator=gen, device="cuda").to(dtype)
    par = np.full((B, R), -1, dtype=np.int32)
    for b, t in enumerate(trees):
        par[b, :len(t)] = t
    par_t = torch.tensor(par, device="cuda")
    f64 = lambda t: t.float().cpu().numpy().astype(np.float64)
    depths = [_depths(t) for t in trees]
    tol_max, tol_mean, tol_lse = (2e-2, 2e-3, 2e-3) if dtype == torch.bfloat16 else (1e-4, 1e-5, 1e-5)
    for depth in range(1, max(max(x) for x in depths) + 1):
        # realized nodes so far and the first node of this depth, per sequence
        total = [sum(1 for x in dp if x <= depth) for dp in depths]
        q0 = [sum(1 for x in dp if x < depth) for dp in depths]
        nr = torch.tensor(total, dtype=torch.int32, device="cuda")
        q0_t = torch.tensor(q0, dtype=torch.int32, device="cuda")
        mask, _, _, _ = tree_build(par_t, nr, torch.tensor(ctx, device="cuda"))
        out = torch.full_like(q, 7.0)
        lse = torch.full((B, hq, R), 7.0, device="cuda")
        draft_tree_attention(q, kp, vp, torch.tensor(table, device="cuda"), torch.tensor(ctx, device="cuda"), sk, sv,
                             mask, nr, q0_t, d ** -0.5, out=out, lse=lse, kernel=kernel,
                             max_q_nodes=max(t - z for t, z in zip(total, q0)) if depth % 2 else None)
        torch.cuda.synchronize()
        want_o, want_l = O.draft_depth_attention_batch(f64(q), f64(kp), f64(vp), table, ctx, f64(sk), f64(sv),
                                                       [t[:total[b]] for b, t in enumerate(trees)], q0, d ** -0.5)
        got_o, got_l = out.float().cpu().numpy(), lse.cpu().numpy()
        for b in range(B):
            assert (got_o[b, :q0[b]] == 7.0).all() and (got_l[b, :, :q0[b]] == 7.0).all(), (depth, b)
            if q0[b] >= total[b]:
                continue
            e = np.abs(got_o[b, q0[b]:total[b]] - want_o[b, q0[b]:total[b]])
            assert e.max() < tol_max and e.mean() < tol_mean, (depth, b, e.max(), e.mean())
            assert np.abs(got_l[b, :, q0[b]:total[b]] - want_l[b, :, q0[b]:total[b]]).max() < tol_lse, (depth, b)


@pytest.mark.parametrize("B,V,tree", [(4, 128256, "t64"), (1, 4096, "t64"), (3, 1000, "n8"), (2, 4101, "t64")])
def test_attention_fused_greedy_scan(B, V, tree):
    """The greedy argmax scan fused into the attention call (pair kernel's
    idle warp when it runs, else a separate launch) gives the same keys /
    walk as accept_greedy; NaN rows raise the error bit."""
    from paper_2508_08192_b200.sampling import accept_greedy
    from paper_2508_08192_b200.verify import StepInputs, TreeVerifier

    t = TREE64 if tree == "t64" else [-1, -1, 0, 0, 1, 2, 2, 5]
    c = _rand_paged_case(B, 64, 8, 128, 1000, 32, t, seed=B + V)
    R = c["R"]
    rng = np.random.default_rng(V)
    lg = (2.0 * rng.normal(size=(B, R, V))).astype(np.float32)
    lg[:, ::5, 7] = lg[:, ::5, -3] = 40.0  # ties spanning chunks
    am = lg.argmax(-1)
    tok = np.where(rng.random((B, R)) < 0.7, am[:, np.array(c["aug"]).clip(min=0)], rng.integers(V, size=(B, R)))
    tok = torch.tensor(tok.astype(np.int32), device="cuda")
    x = StepInputs(parent=torch.tensor([list(c["aug"])] * B, dtype=torch.int32, device="cuda"), n_rows=c["nr"],
                   ctx_len=c["ctx"], tokens=tok, q=c["q"], tree_k=c["tk"], tree_v=c["tv"],
                   logits=torch.tensor(lg, device="cuda"), k_pool=c["kp"], v_pool=c["vp"], block_table=c["table"])
    for fuse in ("always", False):
        ver = TreeVerifier(scale=128 ** -0.5, fuse_greedy=fuse)
        out, lse, acc, _ = ver.step(x, compact=False)
        ref = accept_greedy(x.logits, x.parent, x.n_rows, x.tokens)
        torch.cuda.synchronize()
        assert int(acc.err[0]) == 0
        assert torch.equal(acc.path_len, ref.path_len) and torch.equal(acc.next_token, ref.next_token)
        for b in range(B):
            n = int(ref.path_len[b])
            assert torch.equal(acc.path[b, :n], ref.path[b, :n])
    x.logits[0, 1, 5] = float("nan")
    ver = TreeVerifier(scale=128 ** -0.5, fuse_greedy="always")
    _, _, acc, _ = ver.step(x, compact=False)
    torch.cuda.synchronize()
    assert int(acc.err[0]) & 2


def test_device_bookkeeping_replays_reference_rounds(golden):
    """Base + draft cache write-back, rewind and block mapping on the device
    allocator, and the hidden tape, over several engine rounds: the logical
    contents equal the reference caches' gathers and tape (bit-exact)."""
    from paper_2508_08192_b200.kvstore import DeviceBlockAllocator, compact_draft_kv, compact_kv, tape_append

    g = golden("bookkeep")
    dev = "cuda"
    for k in range(int(g["n_cases"])):
        p = f"b{k}_"
        bs, hkv, d, n_layers, dim, nb, L = (int(x) for x in g[p + "meta"])
        n_nodes = len(g[p + "parent"])
        mb = nb
        pools = {c: (torch.zeros((n_layers, nb, hkv, bs, d), device=dev), torch.zeros((n_layers, nb, hkv, bs, d),
                                                                                      device=dev))
                 for c in ("base", "draft")}
        alloc = {c: DeviceBlockAllocator(nb, 1, mb, bs, dev) for c in ("base", "draft")}

        def write_rows(c, li, start, kr, vr):
            table = alloc[c].block_table[0].cpu().numpy()
            for j in range(kr.shape[0]):
                pos = start + j
                blk, off = int(table[pos // bs]), pos % bs
                pools[c][0][li, blk, :, off] = _cuda(kr[j].reshape(hkv, d), torch.float32)
                pools[c][1][li, blk, :, off] = _cuda(vr[j].reshape(hkv, d), torch.float32)

        def gather(c, li, n):
            table = alloc[c].block_table[0].cpu().numpy()
            kp, vp = pools[c][0][li].cpu().numpy(), pools[c][1][li].cpu().numpy()
            ks = [kp[table[pos // bs], :, pos % bs].reshape(-1) for pos in range(n)]
            vs = [vp[table[pos // bs], :, pos % bs].reshape(-1) for pos in range(n)]
            return np.stack(ks), np.stack(vs)

        for c, key in (("base", "ib"), ("draft", "id")):
            alloc[c].ensure(_cuda([L - 1], torch.int32))
            for li in range(n_layers):
                write_rows(c, li, 0, g[p + f"{key}{li}"][0], g[p + f"{key}{li}"][1])
        itape = g[p + "itape"]
        cap = itape.shape[0] + int(g[p + "rounds"]) * (n_nodes + 1)
        tape = torch.zeros((1, cap, dim), device=dev)
        tape[0, :itape.shape[0]] = _cuda(itape, torch.float32)
        tape_len = _cuda([itape.shape[0]], torch.int32)
        err = torch.zeros((1,), dtype=torch.int32, device=dev)
        for rd in range(int(g[p + "rounds"])):
            q = f"{p}r{rd}_"
            path = [int(x) for x in g[q + "path"]]
            kept = int(g[q + "kept"])
            for c in ("base", "draft"):
                alloc[c].alloc_for_step(_cuda([L], torch.int32), n_nodes)
            for li in range(n_layers):
                write_rows("draft", li, L - 1, g[q + "align_k"], g[q + "align_v"])
            pt = np.zeros((1, n_nodes + 1), dtype=np.int32)
            pt[0, :len(path)] = path
            pt, plen, nk, ctx = (_cuda(pt, torch.int32), _cuda([len(path)], torch.int32), _cuda([kept], torch.int32),
                                 _cuda([L - 1], torch.int32))
            bk = torch.stack([_cuda(g[q + f"bk{li}"].reshape(n_nodes + 1, hkv, d), torch.float32)
                              for li in range(n_layers)])[:, None]
            bv = torch.stack([_cuda(g[q + f"bv{li}"].reshape(n_nodes + 1, hkv, d), torch.float32)
                              for li in range(n_layers)])[:, None]
            sk = torch.stack([_cuda(g[q + f"sk{li}"].reshape(n_nodes, hkv, d), torch.float32)
                              for li in range(n_layers)])[:, None]
            sv = torch.stack([_cuda(g[q + f"sv{li}"].reshape(n_nodes, hkv, d), torch.float32)
                              for li in range(n_layers)])[:, None]
            compact_kv(bk, bv, pools["base"][0], pools["base"][1], alloc["base"].block_table, ctx, pt, plen, nk)
            compact_draft_kv(sk, sv, pools["draft"][0], pools["draft"][1], alloc["draft"].block_table, ctx, pt, plen,
                             nk)
            tape_append(_cuda(g[q + "hid"][None], torch.float32), tape, tape_len, pt, plen, err, nk)
            L = L + kept
            for c in ("base", "draft"):
                alloc[c].rewind(_cuda([L - 1], torch.int32))
        torch.cuda.synchronize()
        assert L == int(g[p + "final_len"]) and int(err[0]) == 0
        for c in ("base", "draft"):
            alloc[c].check()
        assert [int(alloc[c].n_mapped[0]) for c in ("base", "draft")] == list(g[p + "blocks_used"])
        for li in range(n_layers):
            for c, key in (("base", "gb"), ("draft", "gd")):
                gk, gv = gather(c, li, L - 1)
                np.testing.assert_array_equal(gk, g[p + f"{key}{li}"][0].astype(np.float32))
                np.testing.assert_array_equal(gv, g[p + f"{key}{li}"][1].astype(np.float32))
        np.testing.assert_array_equal(tape[0, :int(tape_len[0])].cpu().numpy(), g[p + "tape"].astype(np.float32))


@pytest.mark.parametrize("chunk,kernel", [(512, 1), (512, 2), (384, 0)])
def test_tree_verify_attention_irope_local_chunk(chunk, kernel):
    """iRoPE local attention: with the tree truncated at
    the chunk boundary (truncate_draft_at_boundary), every row sees prefix
    keys [floor(C / chunk) * chunk, C) -- vs the oracle's LocalChunk mask
    (attention.py:76-84); includes an empty local prefix (C on a boundary).
    chunk 384 is not a tile multiple: the auto path takes the SIMT kernel."""
    from paper_2508_08192_b200.attention import tree_verify_attention
    from paper_2508_08192_b200.drafttree import tree_build

    B, Hq, Hkv, d, bs = 4, 64, 8, 128, 64
    aug = O.augment(tuple(TREE64))
    R = len(aug)
    rng = np.random.default_rng(chunk)
    ctx = np.array([3 * chunk + 17, chunk, 2 * chunk + chunk - 8, 5 * chunk + 100], dtype=np.int32)
    pages = -(-(int(ctx.max()) + R) // bs)
    nb = B * pages + 3
    table = rng.permutation(nb)[:B * pages].reshape(B, pages).astype(np.int32)
    gen = torch.Generator(device="cuda").manual_seed(chunk)
    kp = torch.randn((nb, Hkv, bs, d), generator=gen, device="cuda").to(torch.bfloat16)
    vp = torch.randn((nb, Hkv, bs, d), generator=gen, device="cuda").to(torch.bfloat16)
    q = torch.randn((B, R, Hq, d), generator=gen, device="cuda").to(torch.bfloat16)
    tk = torch.randn((B, R, Hkv, d), generator=gen, device="cuda").to(torch.bfloat16)
    tv = torch.randn((B, R, Hkv, d), generator=gen, device="cuda").to(torch.bfloat16)
    par = torch.tensor([list(aug)] * B, dtype=torch.int32, device="cuda")
    nr = torch.full((B,), R, dtype=torch.int32, device="cuda")
    ctx_t = torch.tensor(ctx, device="cuda")
    mask, _, _, _ = tree_build(par, nr, ctx_t)
    out, lse = tree_verify_attention(q, kp, vp, torch.tensor(table, device="cuda"), ctx_t, tk, tv, mask, nr,
                                     d ** -0.5, kernel=kernel, chunk_len=chunk)
    torch.cuda.synchronize()
    f64 = lambda t: t.float().cpu().numpy().astype(np.float64)
    want_o, want_l = O.tree_verify_attention_batch(f64(q), f64(kp), f64(vp), table, ctx, f64(tk), f64(tv),
                                                   [aug] * B, d ** -0.5, chunk_len=chunk)
    err = np.abs(out.float().cpu().numpy() - want_o)
    assert err.max() < 2e-2 and err.mean() < 2e-3, (err.max(), err.mean())
    assert np.abs(lse.cpu().numpy() - want_l).max() < 2e-3


@pytest.mark.parametrize("mode", ["greedy", "stochastic"])
def test_verifier_step_mixed_batch_edge_cases(mode):
    """One TreeVerifier step over a batch mixing the live edge cases of
    SURVEY 8(a) a2: a root-only tree (R = 1, the non-speculative / truncated
    round), an empty prefix (C = 0), the 8-node tree, the 64-row EAGLE tree
    and a chain; 70B head shapes through the tcgen05 path.  Attention vs the
    float64 oracle, acceptance and compaction exact."""
    from paper_2508_08192_b200.sampling import device_uniforms
    from paper_2508_08192_b200.verify import StepInputs, TreeVerifier

    trees = [O.augment(()), O.augment((-1, -1, 0, 0, 1, 2, 2, 5)), O.augment(tuple(TREE64)), O.augment((-1, 0, 1)),
             O.augment((-1, -1, 0))]
    ctx = np.array([300, 0, 1029, 77, 4096], dtype=np.int32)
    B, Hq, Hkv, d, bs, V, T, top_p = len(trees), 64, 8, 128, 64, 1000, 1.0, 0.9
    R = max(len(t) for t in trees)
    rng = np.random.default_rng(17)
    nbl = [-(-(int(c) + R) // bs) for c in ctx]
    nb = sum(nbl) + 2
    perm = rng.permutation(nb).astype(np.int32)
    table = np.zeros((B, max(nbl)), dtype=np.int32)
    o = 0
    for b in range(B):
        table[b, :nbl[b]] = perm[o:o + nbl[b]]
        o += nbl[b]
    gen = torch.Generator(device="cuda").manual_seed(17)
    rb = lambda *s: torch.randn(*s, generator=gen, device="cuda").to(torch.bfloat16)
    k_pool, v_pool = rb(nb, Hkv, bs, d), rb(nb, Hkv, bs, d)
    q, tk, tv = rb(B, R, Hq, d), rb(B, R, Hkv, d), rb(B, R, Hkv, d)
    par = np.full((B, R), -1, dtype=np.int32)
    nr = np.array([len(t) for t in trees], dtype=np.int32)
    for b, t in enumerate(trees):
        par[b, :len(t)] = t
    tl = (2.0 * rng.normal(size=(B, R, V))).astype(np.float32)
    dl = (tl + 0.5 * rng.normal(size=(B, R, V))).astype(np.float32)
    tokens = np.zeros((B, R), dtype=np.int32)
    for b, t in enumerate(trees):
        for i in range(1, len(t)):
            if mode == "greedy":
                tokens[b, i] = int(np.argmax(tl[b, t[i]])) if rng.random() < 0.6 else int(rng.integers(V))
            else:
                tokens[b, i] = int(O.sample_from(O.target_dist(dl[b, t[i]].astype(np.float64), T, 1.0), rng.random()))
    seeds = torch.arange(B, dtype=torch.int64, device="cuda") + 5
    steps = torch.full((B,), 8, dtype=torch.int64, device="cuda")
    kp0 = k_pool.float().cpu().numpy().astype(np.float64)
    x = StepInputs(parent=torch.tensor(par, device="cuda"), n_rows=torch.tensor(nr, device="cuda"),
                   ctx_len=torch.tensor(ctx, device="cuda"), tokens=torch.tensor(tokens, device="cuda"), q=q,
                   tree_k=tk, tree_v=tv, logits=torch.tensor(tl, device="cuda"), k_pool=k_pool.contiguous(),
                   v_pool=v_pool.contiguous(), block_table=torch.tensor(table, device="cuda"),
                   draft_logits=torch.tensor(dl, device="cuda"), seeds=seeds, steps=steps)
    ver = TreeVerifier(scale=d ** -0.5, temperature=0.0 if mode == "greedy" else T,
                       top_p=1.0 if mode == "greedy" else top_p)
    out, lse, acc, terr = ver.step(x)
    uni = device_uniforms(seeds, steps, R).cpu().numpy()
    torch.cuda.synchronize()
    assert int(terr.abs().sum()) == 0 and int(acc.err[0]) == 0
    f64 = lambda t_: t_.float().cpu().numpy().astype(np.float64)
    want_o, want_l = O.tree_verify_attention_batch(f64(q), kp0, f64(v_pool), table, ctx, f64(tk), f64(tv),
                                                   [tuple(t) for t in trees], d ** -0.5)
    got_o, got_l = out.float().cpu().numpy(), lse.cpu().numpy()
    for b in range(B):
        n = nr[b]
        assert np.abs(got_o[b, :n] - want_o[b, :n]).max() < 2e-2, b
        assert np.abs(got_l[b, :, :n] - want_l[b, :, :n]).max() < 2e-3, b
        raw = tuple(p - 1 if p > 0 else -1 for p in trees[b][1:])
        if mode == "greedy":
            path, nxt, used = O.greedy_walk(raw, tokens[b, 1:], np.argmax(tl[b].astype(np.float64), axis=1))
        else:
            tdists = [O.target_dist(tl[b, r].astype(np.float64), T, top_p) for r in range(n)]
            nd = [O.target_dist(dl[b, trees[b][i]].astype(np.float64), T, 1.0) for i in range(1, n)]
            path, nxt, _res, used = O.mss_verify(raw, tokens[b, 1:], nd, tdists, uni[b])
        plen = int(acc.path_len[b])
        assert acc.path[b, :plen].cpu().tolist() == list(path), (b, mode)
        assert int(acc.next_token[b]) == nxt and int(acc.uniforms_used[b]) == used, (b, mode)
        O.compact_kv(kp0, kp0.copy(), table[b], int(ctx[b]), f64(tk)[b], f64(tv)[b], list(path), plen + 1)
    np.testing.assert_array_equal(x.k_pool.float().cpu().numpy(), kp0.astype(np.float32))


def test_tcgen05_r65_variant_vs_oracle():
    """The mandatory R = 65 variant (64 drafts: TREE64 + a 7th child of node
    0, not breadth-first) at 70B shapes: 520 query rows per KV head = three
    256-row pair tiles, the last one 8 rows deep."""
    from paper_2508_08192_b200.attention import tree_verify_attention

    c = _rand_paged_case(2, 64, 8, 128, 3000, 64, TREE64 + [0], seed=65)
    assert c["R"] == 65
    out, lse = tree_verify_attention(c["q"], c["kp"], c["vp"], c["table"], c["ctx"], c["tk"], c["tv"], c["mask"],
                                     c["nr"], 128 ** -0.5, kernel=1)
    torch.cuda.synchronize()
    f64 = lambda t: t.float().cpu().numpy().astype(np.float64)
    want_o, want_l = O.tree_verify_attention_batch(f64(c["q"]), f64(c["kp"]), f64(c["vp"]), c["table_np"],
                                                   c["ctx_np"], f64(c["tk"]), f64(c["tv"]), [c["aug"]] * 2,
                                                   128 ** -0.5)
    err = np.abs(out.float().cpu().numpy() - want_o)
    assert err.max() < 2e-2 and err.mean() < 2e-3, (err.max(), err.mean())
    assert np.abs(lse.cpu().numpy() - want_l).max() < 2e-3


@pytest.mark.parametrize("hq,splits,plant", [(64, 0, False), (64, 148, False), (64, 5, False), (32, 0, False),
                                              (32, 148, False), (64, 0, True), (64, 148, True)])
def test_tcgen05_fused_tail_rows_vs_oracle(hq, splits, plant, monkeypatch):
    """R = 65 on the pair kernel with SDB_ATTN_TAIL=1 (off by default: exact
    but slower): the rows past the last full 256-row
    block (g = 8: node 64's 8 heads; g = 4: 4 rows) ride along in that
    block's units (warps 2 / 3, N = 16 S^T and O^T MMAs, per-CTA key halves
    merged at the unit end).  Whole units, stream-K pieces merged by the
    fix-up (148 and 5 workers), and a planted key ~170 nats above the tail
    rows' reference (their exact recompute) against the float64 oracle."""
    from paper_2508_08192_b200.attention import tree_verify_attention

    monkeypatch.setenv("SDB_ATTN_TAIL", "1")

    c = _rand_paged_case(2, hq, 8, 128, 3000, 64, TREE64 + [0], seed=650 + hq + splits)
    assert c["R"] == 65
    g = hq // 8
    if plant:
        kvh, j = 5, 2800
        j = min(j, int(c["ctx_np"][1]) - 1)
        page = int(c["table_np"][1, j // 64])
        c["kp"][page, kvh, j % 64, :] = 4.0
        c["q"][1, 64, kvh * g:(kvh + 1) * g, :] = 4.0
    out, lse = tree_verify_attention(c["q"], c["kp"], c["vp"], c["table"], c["ctx"], c["tk"], c["tv"], c["mask"],
                                     c["nr"], 128 ** -0.5, num_splits=splits, kernel=1)
    torch.cuda.synchronize()
    f64 = lambda t: t.float().cpu().numpy().astype(np.float64)
    want_o, want_l = O.tree_verify_attention_batch(f64(c["q"]), f64(c["kp"]), f64(c["vp"]), c["table_np"],
                                                   c["ctx_np"], f64(c["tk"]), f64(c["tv"]), [c["aug"]] * 2,
                                                   128 ** -0.5)
    got_o = out.float().cpu().numpy()
    assert np.isfinite(got_o).all()
    err = np.abs(got_o - want_o)
    assert err.max() < 2e-2 and err.mean() < 2e-3, (err.max(), err.mean())
    tail = np.abs(got_o[:, 64] - want_o[:, 64])
    assert tail.max() < 2e-2, tail.max()
    assert np.abs(lse.cpu().numpy() - want_l).max() < 2e-3
    if plant:
        assert want_l[1, kvh * g:(kvh + 1) * g, 64].min() > 150


@pytest.mark.parametrize("tree", ["tree64", "chain3"])
@pytest.mark.parametrize("ctas", [0, 148])
def test_tcgen05_fixed_reference_overflow_exact(ctas, tree):
    """The tcgen05 softmax takes each unit piece's first-tile row max as a
    fixed reference (no max pass, no rescale afterwards): the pair kernel
    (64-row tree) and the 1-CTA kernel with one query tile (chain-3: 32 rows
    per KV head, two S slots).  A key whose score lies ~170 nats above
    everything in the first tile (exp2 would overflow against that reference)
    sends the affected rows through the exact recompute; whole units (ctas 0)
    and stream-K pieces merged by the fix-up (ctas 148 at B = 1) must both
    match the float64 oracle."""
    from paper_2508_08192_b200.attention import tree_verify_attention

    B = 2 if ctas == 0 else 1
    parents = TREE64 if tree == "tree64" else (-1, 0, 1)
    c = _rand_paged_case(B, 64, 8, 128, 3000, 64, parents, seed=91, ragged=False)
    kvh, g, j = 3, 8, 2500  # late prefix key of sequence 0 / KV head 3
    page = int(c["table_np"][0, j // 64])
    c["kp"][page, kvh, j % 64, :] = 4.0
    c["q"][0, :, kvh * g:(kvh + 1) * g, :] = 4.0
    out, lse = tree_verify_attention(c["q"], c["kp"], c["vp"], c["table"], c["ctx"], c["tk"], c["tv"], c["mask"],
                                     c["nr"], 128 ** -0.5, num_splits=ctas, kernel=1)
    torch.cuda.synchronize()
    f64 = lambda t: t.float().cpu().numpy().astype(np.float64)
    want_o, want_l = O.tree_verify_attention_batch(f64(c["q"]), f64(c["kp"]), f64(c["vp"]), c["table_np"],
                                                   c["ctx_np"], f64(c["tk"]), f64(c["tv"]), [c["aug"]] * B,
                                                   128 ** -0.5)
    got_o = out.float().cpu().numpy()
    assert np.isfinite(got_o).all()
    err = np.abs(got_o - want_o)
    assert err.max() < 2e-2 and err.mean() < 2e-3, (err.max(), err.mean())
    assert np.abs(lse.cpu().numpy() - want_l).max() < 2e-3
    # the flagged rows really are dominated by the planted key (LSE ~ 181 nats)
    assert want_l[0, kvh * g:(kvh + 1) * g].min() > 150
