"""Pin the CPU oracle to the reference's own outputs (tests/golden, produced by
oracle/make_golden.py from the unmodified reference) and to the reference
test suite's known answers.  CPU only."""

import numpy as np
import pytest

from oracle import specdec_oracle as O


def _parents(row, n):
    return tuple(int(x) for x in row[:n])


def test_tree_structures_match_reference(golden):
    g = golden("trees")
    for i in range(len(g["n_rows"])):
        n = int(g["n_rows"][i])
        raw = _parents(g["raw_parent"][i], int(g["raw_len"][i]))
        aug = O.augment(raw)
        assert aug == _parents(g["parent_aug"][i], n)
        np.testing.assert_array_equal(O.suffix_mask(aug), g["mask"][i, :n, :n])
        np.testing.assert_array_equal(O.tree_depth(aug), g["depth"][i, :n])
        np.testing.assert_array_equal(O.positions(aug, int(g["ctx"][i])), g["pos"][i, :n])


def test_tree_validation_matches_reference(golden):
    g = golden("trees")
    for i, ok in enumerate(g["bad_valid"]):
        p = _parents(g["bad_parent"][i], int(g["bad_len"][i]))
        if ok:
            O.tree_depth(p)
        else:
            with pytest.raises(O.OracleError):
                O.tree_depth(p)


def test_mask_word_known_answers():
    # full:2,2 augmented and the reference N8 tree
    full22 = O.augment((-1, -1, 0, 0, 1, 1))
    words = O.mask_words(O.suffix_mask(full22))[:, 0]
    assert list(words) == [1, 3, 5, 11, 19, 37, 69]
    n8 = O.augment((-1, -1, 0, 0, 1, 2, 2, 5))
    assert list(O.mask_words(O.suffix_mask(n8))[:, 0]) == [1, 3, 5, 11, 19, 37, 75, 139, 331]


def test_tree_attention_f64_matches_reference(golden):
    g = golden("attention_f64")
    for ci in range(int(g["n_cases"])):
        p = f"c{ci}_"
        nh, hd, ctx, chunk = (int(x) for x in g[p + "meta"])
        parent = tuple(int(x) for x in g[p + "parent"])
        out, lse = O.tree_attention(g[p + "q"], g[p + "ck"], g[p + "cv"], g[p + "tk"], g[p + "tv"],
                                    parent, hd ** -0.5, nh, chunk_len=None if chunk < 0 else chunk)
        np.testing.assert_allclose(out, g[p + "out"], atol=1e-12, rtol=0)
        np.testing.assert_allclose(lse, g[p + "lse"], atol=1e-12, rtol=0)


def test_attend_and_merge_match_reference(golden):
    g = golden("attend_merge")
    q, k, v = g["q"], g["k"], g["v"]
    a = O.attend(q, k[:3], v[:3], None, 0.3, 2)
    b = O.attend(q, k[3:], v[3:], None, 0.3, 2)
    np.testing.assert_allclose(a[0], g["a_out"], atol=1e-13)
    np.testing.assert_allclose(b[1], g["b_lse"], atol=1e-13)
    m = O.merge_partials([a, b], 2)
    np.testing.assert_allclose(m[0], g["m_out"], atol=1e-13)
    np.testing.assert_allclose(m[1], g["m_lse"], atol=1e-13)
    e = O.attend(q, np.zeros((0, 8)), np.zeros((0, 8)), None, 0.3, 2)
    np.testing.assert_array_equal(e[0], g["e_out"])
    np.testing.assert_array_equal(e[1], g["e_lse"])
    c = O.attend(q, k, v, g["mask"], 0.3, 2)
    np.testing.assert_allclose(c[0], g["c_out"], atol=1e-13)
    np.testing.assert_array_equal(np.isinf(c[1]), np.isinf(g["c_lse"]))
    with pytest.raises(O.OracleError):
        O.merge_partials([e, e], 2)


def test_gqa_paged_attention_matches_reference(golden):
    g = golden("attention_gqa")
    for name in g["names"]:
        p = str(name) + "_"
        bsz, hq, hkv, d, bs, r_max = (int(x) for x in g[p + "meta"])
        parents = [_parents(g[p + "parent_aug"][b], int(g[p + "n_rows"][b])) for b in range(bsz)]
        out, lse = O.tree_verify_attention_batch(
            g[p + "q"].astype(np.float64), g[p + "k_pool"].astype(np.float64),
            g[p + "v_pool"].astype(np.float64), g[p + "table"], g[p + "ctx"],
            g[p + "tk"].astype(np.float64), g[p + "tv"].astype(np.float64), parents, d ** -0.5)
        np.testing.assert_allclose(out, g[p + "out"], atol=1e-12)
        np.testing.assert_allclose(lse, g[p + "lse"], atol=1e-12)


def test_greedy_walk_equals_reference_mss(golden):
    g = golden("accept_greedy")
    for k in range(int(g["n_cases"])):
        p = f"g{k}_"
        parent = tuple(int(x) for x in g[p + "parent"])
        am = np.argmax(g[p + "logits"].astype(np.float64), axis=1)
        path, nxt, used = O.greedy_walk(parent, g[p + "tokens"], am)
        assert path == list(g[p + "path"])
        assert nxt == int(g[p + "next"])
        assert used == int(g[p + "used"])


def test_stochastic_mss_matches_reference(golden):
    g = golden("accept_stochastic")
    for k in range(int(g["n_cases"])):
        p = f"s{k}_"
        temp, top_p, _seed = g[p + "meta"]
        parent = tuple(int(x) for x in g[p + "parent"])
        logits, dl = g[p + "logits"], g[p + "draft_logits"]
        qd = [O.target_dist(dl[0 if a == -1 else 1 + a], temp, 1.0) for a in parent]
        dists = [O.target_dist(logits[i], temp, top_p) for i in range(len(parent) + 1)]
        np.testing.assert_allclose(dists[0], g[p + "dist0"], atol=1e-15)
        path, nxt, resid, used = O.mss_verify(parent, g[p + "tokens"], qd, dists, g[p + "uniforms"])
        assert path == list(g[p + "path"])
        assert nxt == int(g[p + "next"])
        assert used == int(g[p + "used"])
        np.testing.assert_allclose(resid, g[p + "residual"], atol=1e-15)
        # the lazy accessor form (rows computed on demand) walks identically
        lz = O.mss_verify(parent, g[p + "tokens"], lambda c: qd[c],
                          lambda i: O.target_dist(logits[i], temp, top_p), g[p + "uniforms"])
        assert lz[0] == path and lz[1] == nxt and lz[3] == used
        np.testing.assert_array_equal(lz[2], resid)


def test_sampling_known_answers(golden):
    g = golden("sampling_kat")
    for i in range(len(g["ps"])):
        np.testing.assert_allclose(O.top_p_mask(g["dists"][i], g["ps"][i]), g["top_p"][i], atol=1e-15)
        assert O.sample_from(g["dists"][i], g["us"][i]) == int(g["sample"][i])
    # reference tests/test_sampling.py:11-58 known answers
    d = np.array([0.5, 0.3, 0.2])
    np.testing.assert_allclose(O.top_p_mask(d, 0.8), [0.625, 0.375, 0.0])
    np.testing.assert_allclose(O.top_p_mask(d, 0.51), [0.625, 0.375, 0.0])
    np.testing.assert_allclose(O.top_p_mask(np.full(4, 0.25), 0.5), [0.5, 0.5, 0.0, 0.0])
    np.testing.assert_array_equal(O.target_dist(np.array([0.1, 3.0, -1.0]), 0.0, 1.0), [0, 1, 0])
    d = np.array([0.2, 0.5, 0.3])
    assert [O.sample_from(d, u) for u in (0.0, 0.19, 0.2, 0.69, 0.7, 0.999999)] == [0, 0, 1, 1, 2, 2]


def test_mss_known_answers():
    # reference tests/test_sampling.py:79-138
    q = np.array([0.5, 0.5, 0.0])
    p = np.array([0.6, 0.4, 0.0])
    r = O.mss_verify((-1, 0), [0, 0], [q, q], [p, p, np.array([0.0, 0.0, 1.0])], [0.9, 0.9, 0.5])
    assert r[0] == [0, 1] and r[1] == 2 and r[3] == 3
    r = O.mss_verify((-1,), [0], [np.array([1.0, 0.0])], [np.array([0.3, 0.7])] * 2, [0.5, 0.0])
    assert r[0] == [] and r[1] == 1
    q1 = np.array([1.0, 0.0, 0.0])
    r = O.mss_verify((-1, -1), [0, 1], [q1, q1], [np.array([0.0, 1.0, 0.0])] * 3, [0.5] * 3)
    assert r[0] == [1] and r[1] == 1
    r = O.mss_verify((-1,), [0], [np.array([1.0, 0.0])], [np.array([1.0, 0.0])] * 2, [1.0, 0.3])
    assert r[0] == [] and r[1] == 0
    with pytest.raises(O.OracleError):
        O.mss_verify((-1,), [0], [np.array([0.5, 0.5])], [np.array([0.5, 0.5])] * 2, [0.5])


def test_philox_matches_reference(golden):
    g = golden("philox")
    for i in range(int(g["n"])):
        seed, step, b, w = (int(x) for x in g[f"p{i}_spec"])
        np.testing.assert_array_equal(O.rank_sliced_uniforms(seed, step, b, w), g[f"p{i}_u"])
    assert O.rank_sliced_uniforms(0, 0, 1, 5)[0, 0] == 0.011546754286331562


def test_compaction_matches_reference_cache(golden):
    g = golden("compact")
    for k in range(int(g["n_cases"])):
        p = f"k{k}_"
        bs, L, hkv, d, n_layers, nb, kept = (int(x) for x in g[p + "meta"])
        table = g[p + "table"]
        path = [int(x) for x in g[p + "path"]]
        for li in range(n_layers):
            kp = np.zeros((nb, hkv, bs, d))
            vp = np.zeros((nb, hkv, bs, d))
            C = L - 1
            O.paged_write(kp, table, 0, g[p + f"ck{li}"])
            O.paged_write(vp, table, 0, g[p + f"cv{li}"])
            tk = g[p + f"tk{li}"].reshape(-1, hkv, d)
            tv = g[p + f"tv{li}"].reshape(-1, hkv, d)
            O.compact_kv(kp, vp, table, C, tk, tv, path, kept)
            n = L + kept - 1
            np.testing.assert_array_equal(O.paged_gather(kp, table, n), g[p + f"gk{li}"])
            np.testing.assert_array_equal(O.paged_gather(vp, table, n), g[p + f"gv{li}"])


def test_draft_depth_attention_matches_reference(golden):
    """Oracle of the draft stage's depth step (rectangular suffix mask over
    carried ++ new K/V, engine.py:424-432) vs the reference's attend /
    merge on the engine's own vis-row masks."""
    g = golden("draft_attention")
    for k in range(int(g["n_cases"])):
        p = f"d{k}_"
        hq, hkv, d, ctx, q0, total = (int(x) for x in g[p + "meta"])
        # the vis rows the engine builds equal the realized tree's ancestor closure
        parent = tuple(int(x) for x in g[p + "parent"])[:total]
        np.testing.assert_array_equal(g[p + "mask"], O.suffix_mask(parent)[q0:total])
        out, lse = O.draft_depth_attention(g[p + "q"], g[p + "ck"], g[p + "cv"], g[p + "sk"], g[p + "sv"],
                                           g[p + "mask"], d ** -0.5, hq, hkv)
        np.testing.assert_allclose(out, g[p + "out"], atol=1e-12)
        np.testing.assert_allclose(lse, g[p + "lse"], atol=1e-12)


def test_bookkeeping_replay_matches_reference(golden):
    """Several rounds of base + draft cache write-back / rewind and the
    hidden tape (engine.py:504-533) on logical rows == the reference caches'
    gathers and tape."""
    g = golden("bookkeep")
    for k in range(int(g["n_cases"])):
        p = f"b{k}_"
        bs, hkv, d, n_layers, dim, nb, L = (int(x) for x in g[p + "meta"])
        base = [[list(g[p + f"ib{li}"][0]), list(g[p + f"ib{li}"][1])] for li in range(n_layers)]
        draft = [[list(g[p + f"id{li}"][0]), list(g[p + f"id{li}"][1])] for li in range(n_layers)]
        tape = list(g[p + "itape"])
        for rd in range(int(g[p + "rounds"])):
            q = f"{p}r{rd}_"
            L = O.bookkeep_round(base, draft, tape, L, list(g[q + "path"]), int(g[q + "kept"]),
                                 [(g[q + f"bk{li}"], g[q + f"bv{li}"]) for li in range(n_layers)],
                                 [(g[q + f"sk{li}"], g[q + f"sv{li}"]) for li in range(n_layers)], g[q + "hid"],
                                 [(g[q + "align_k"][0], g[q + "align_v"][0])] * n_layers)
        assert L == int(g[p + "final_len"])
        for li in range(n_layers):
            np.testing.assert_array_equal(np.stack(base[li][0]), g[p + f"gb{li}"][0])
            np.testing.assert_array_equal(np.stack(base[li][1]), g[p + f"gb{li}"][1])
            np.testing.assert_array_equal(np.stack(draft[li][0]), g[p + f"gd{li}"][0])
            np.testing.assert_array_equal(np.stack(draft[li][1]), g[p + f"gd{li}"][1])
        np.testing.assert_array_equal(np.stack(tape), g[p + "tape"])
