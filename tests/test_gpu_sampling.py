"""GPU parity of the sampling side of the path: the device Philox stream vs
the reference's rank_sliced_uniforms, and stochastic (T > 0) acceptance at the
full Llama-3 vocabulary vs the CPU oracle (target_dist + mss_verify in
float64).  Needs a B200."""

import numpy as np
import pytest

torch = pytest.importorskip("torch")

pytestmark = pytest.mark.gpu

from oracle import specdec_oracle as O  # noqa: E402

TREE64 = [-1, -1, -1, -1, -1, -1, -1, -1, 0, 0, 0, 0, 0, 0, 1, 1, 1, 1, 1, 2, 2, 2, 2, 3, 3, 3, 4, 4, 5, 5, 6, 7,
          8, 8, 8, 8, 9, 9, 9, 10, 10, 10, 11, 11, 12, 13, 14, 15, 32, 32, 32, 33, 33, 34, 34, 35, 36, 37, 48, 48, 49,
          50, 51]


@pytest.fixture(scope="module", autouse=True)
def _lib_loaded():
    from paper_2508_08192_b200 import _lib

    _lib.load()


def _i64(vals):
    # uint64 bit patterns as int64
    return torch.tensor(np.array(vals, dtype=np.uint64).view(np.int64), device="cuda")


def test_device_philox_matches_reference_golden(golden):
    from paper_2508_08192_b200.sampling import device_uniforms

    g = golden("philox")
    for i in range(int(g["n"])):
        seed, step, b, w = (int(x) for x in g[f"p{i}_spec"])
        want = g[f"p{i}_u"]
        for row in range(b):
            got = device_uniforms(_i64([seed]), _i64([step]), w, row=row).cpu().numpy()[0]
            np.testing.assert_array_equal(got, want[row])
    got = device_uniforms(_i64([0]), _i64([0]), 5).cpu().numpy()
    assert got[0, 0] == 0.011546754286331562


def test_device_philox_batch_of_sessions_vs_oracle():
    """One launch for a batch of sessions at different (seed, step); large
    uint64 seeds; widths that are not multiples of 4; rows > 0."""
    from paper_2508_08192_b200.sampling import device_uniforms

    rng = np.random.default_rng(5)
    seeds = [int(x) for x in rng.integers(0, 2**63, size=6, dtype=np.int64)] + [2**64 - 1, 0]
    steps = [2 * int(r) + 2 for r in rng.integers(0, 1000, size=8)]
    for width, row in ((65, 0), (64, 0), (7, 3), (1, 11), (130, 2)):
        got = device_uniforms(_i64(seeds), _i64(steps), width, row=row).cpu().numpy()
        for b in range(len(seeds)):
            want = O.rank_sliced_uniforms(seeds[b], steps[b], row + 1, width)[row]
            np.testing.assert_array_equal(got[b], want)


def _stochastic_case(B, V, tree, temperature, top_p, seed):
    """Synthetic inputs of SURVEY 8(d): target N(0, 2^2), draft = target +
    N(0, 0.5^2), node tokens sampled from the parent's draft q (stochastic
    drafting, engine.py:393-394), uniforms from the reference Philox."""
    rng = np.random.default_rng(seed)
    aug = O.augment(tuple(tree))
    R = len(aug)
    tl = (2.0 * rng.normal(size=(B, R, V))).astype(np.float32)
    dl = (tl + 0.5 * rng.normal(size=(B, R, V))).astype(np.float32)
    tokens = np.zeros((B, R), dtype=np.int32)
    for b in range(B):
        for i in range(1, R):
            q = O.target_dist(dl[b, aug[i]].astype(np.float64), temperature, 1.0)
            tokens[b, i] = int(O.sample_from(q, rng.random()))
    seeds = [1234 + b for b in range(B)]
    steps = [2 * (b + 3) + 2 for b in range(B)]
    return aug, tl, dl, tokens, seeds, steps


def _oracle_accept(aug, tl, dl, tokens, uniforms, temperature, top_p):
    parent = tuple(p - 1 if p > 0 else -1 for p in aug[1:])
    tdists = [O.target_dist(tl[r].astype(np.float64), temperature, top_p) for r in range(len(aug))]
    qcache = {}
    ndists = []
    for i, p in enumerate(aug[1:], 1):
        if p not in qcache:
            qcache[p] = O.target_dist(dl[p].astype(np.float64), temperature, 1.0)
        ndists.append(qcache[p])
    return O.mss_verify(parent, tokens[1:], ndists, tdists, uniforms)


@pytest.mark.parametrize("top_p,lazy,walk_cl", [(0.9, True, None), (0.9, False, None), (1.0, True, None),
                                                 (0.9, True, "4"), (0.9, False, "2")])
def test_accept_stochastic_full_vocab_vs_oracle(top_p, lazy, walk_cl, monkeypatch):
    """Llama-3 vocabulary (128,256), the 64-row EAGLE tree, uniforms drawn on
    the device from (seed, step): path, next token and uniforms_used must
    equal the float64 oracle's (lazy walk and eager every-row reduction).
    walk_cl forces the walk's cluster width: 4 and 2 give vocabulary slices
    too wide for the shared-memory bonus values, and at 2 the nucleus
    overflows the shared-memory compaction list (full-row passes)."""
    from paper_2508_08192_b200.sampling import StochasticAcceptor

    if walk_cl:
        monkeypatch.setenv("SDB_WALK_CL", walk_cl)

    def accept_stochastic(*a, **k):
        return StochasticAcceptor(lazy=lazy)(*a, **k)

    B, V, T = 3, 128256, 1.0
    aug, tl, dl, tokens, seeds, steps = _stochastic_case(B, V, TREE64, T, top_p, seed=11)
    R = len(aug)
    par = torch.tensor([aug] * B, dtype=torch.int32, device="cuda")
    res = accept_stochastic(torch.tensor(tl, device="cuda"), torch.tensor(dl, device="cuda"), T, top_p, par,
                            torch.full((B,), R, dtype=torch.int32, device="cuda"),
                            torch.tensor(tokens, device="cuda"), seeds=_i64(seeds), steps=_i64(steps))
    torch.cuda.synchronize()
    assert int(res.err[0]) == 0
    for b in range(B):
        uni = O.rank_sliced_uniforms(seeds[b], steps[b], 1, R)[0]
        path, nxt, _res, used = _oracle_accept(aug, tl[b], dl[b], tokens[b], uni, T, top_p)
        plen = int(res.path_len[b])
        assert res.path[b, :plen].cpu().tolist() == list(path), b
        assert int(res.next_token[b]) == nxt and int(res.uniforms_used[b]) == used, b


@pytest.mark.parametrize("top_p,lazy", [(0.9, True), (0.9, False), (1.0, True)])
def test_accept_stochastic_odd_vocab_vs_oracle(top_p, lazy):
    """V = 4099 (rows not 16-byte aligned): the scalar paths of the row
    stats, the walk's nucleus compaction and the bonus pass."""
    from paper_2508_08192_b200.sampling import StochasticAcceptor

    B, V, T = 3, 4099, 0.9
    aug, tl, dl, tokens, seeds, steps = _stochastic_case(B, V, TREE64, T, top_p, seed=41)
    R = len(aug)
    par = torch.tensor([aug] * B, dtype=torch.int32, device="cuda")
    res = StochasticAcceptor(lazy=lazy)(torch.tensor(tl, device="cuda"), torch.tensor(dl, device="cuda"), T, top_p,
                                        par, torch.full((B,), R, dtype=torch.int32, device="cuda"),
                                        torch.tensor(tokens, device="cuda"), seeds=_i64(seeds), steps=_i64(steps))
    torch.cuda.synchronize()
    assert int(res.err[0]) == 0
    for b in range(B):
        uni = O.rank_sliced_uniforms(seeds[b], steps[b], 1, R)[0]
        path, nxt, _res, used = _oracle_accept(aug, tl[b], dl[b], tokens[b], uni, T, top_p)
        plen = int(res.path_len[b])
        assert res.path[b, :plen].cpu().tolist() == list(path), b
        assert int(res.next_token[b]) == nxt and int(res.uniforms_used[b]) == used, b


def test_lazy_walk_repeatable_at_full_occupancy():
    """64 sequences (8-CTA clusters in two waves, the validation scan on a
    second stream): 25 repeated calls give identical results (the cluster
    CTAs share the lazy state; a race shows up as a mismatch or a fault)."""
    from paper_2508_08192_b200.sampling import StochasticAcceptor, tree_levels

    B, V = 64, 32768
    g = torch.Generator(device="cuda").manual_seed(5)
    aug = O.augment(tuple(TREE64))
    R = len(aug)
    tl = torch.randn((B, R, V), generator=g, device="cuda") * 2.0
    dl = tl + 0.5 * torch.randn((B, R, V), generator=g, device="cuda")
    tok = torch.randint(0, V, (B, R), generator=g, device="cuda", dtype=torch.int32)
    par = torch.tensor([aug] * B, dtype=torch.int32, device="cuda")
    nr = torch.full((B,), R, dtype=torch.int32, device="cuda")
    seeds = torch.arange(B, dtype=torch.int64, device="cuda") + 77
    steps = torch.full((B,), 6, dtype=torch.int64, device="cuda")
    acc = StochasticAcceptor(lazy=True, levels=tree_levels(par))

    def run():
        r = acc(tl, dl, 1.0, 0.9, par, nr, tok, seeds=seeds, steps=steps)
        return [t.clone() for t in (r.path, r.path_len, r.next_token, r.uniforms_used, r.err)]

    ref = run()
    for _ in range(25):
        got = run()
        assert all(torch.equal(a, b) for a, b in zip(ref, got))
    assert int(ref[4][0]) == 0


@pytest.mark.parametrize("lazy", [True, False])
def test_accept_stochastic_wide_tree_vs_oracle(lazy):
    """A 599-wide root (603 rows): the walk gathers a node's children a
    512-row window at a time, so the decisions cross a window boundary.  The
    first 550 root children carry a token outside the top-p nucleus (p = 0:
    always rejected, the residual keeps shrinking by q), the rest are drawn
    from the draft q; three children hang below draft node 0."""
    from paper_2508_08192_b200.sampling import StochasticAcceptor

    B, V, T, top_p = 2, 512, 1.0, 0.5
    tree = [-1] * 599 + [0] * 3
    aug, tl, dl, tokens, seeds, steps = _stochastic_case(B, V, tree, T, top_p, seed=31)
    R = len(aug)
    for b in range(B):
        tokens[b, 1:551] = int(np.argmin(tl[b, 0]))  # lowest target logit: outside the nucleus
    par = torch.tensor([aug] * B, dtype=torch.int32, device="cuda")
    res = StochasticAcceptor(lazy=lazy)(torch.tensor(tl, device="cuda"), torch.tensor(dl, device="cuda"), T, top_p,
                                        par, torch.full((B,), R, dtype=torch.int32, device="cuda"),
                                        torch.tensor(tokens, device="cuda"), seeds=_i64(seeds), steps=_i64(steps))
    torch.cuda.synchronize()
    assert int(res.err[0]) == 0
    for b in range(B):
        uni = O.rank_sliced_uniforms(seeds[b], steps[b], 1, R)[0]
        path, nxt, _res, used = _oracle_accept(aug, tl[b], dl[b], tokens[b], uni, T, top_p)
        assert used > 551, used  # the decisions did cross the first window
        plen = int(res.path_len[b])
        assert res.path[b, :plen].cpu().tolist() == list(path), b
        assert int(res.next_token[b]) == nxt and int(res.uniforms_used[b]) == used, b


# ---------------------------------------------------------------------------
# vocab-sharded stochastic acceptance: every rank's kernels run
# in this process (VirtualComm); the protocol is the one torch.distributed runs
# ---------------------------------------------------------------------------

def _dev(x, dt):
    return torch.as_tensor(np.ascontiguousarray(x)).to(device="cuda", dtype=dt)


def test_sharded_stochastic_matches_reference_golden(golden):
    """Reference golden MSS cases (V = 2048, several temperatures / top-p),
    vocab split over 2, 3 and 8 ranks: every rank reports the reference's
    path, bonus token and uniforms_used; residual slices tile the reference
    residual."""
    from paper_2508_08192_b200.sharding import run_virtual_sharded_stochastic

    g = golden("accept_stochastic")
    from test_gpu_parity import _aug_batch

    for world in (2, 3, 8):
        for k in range(int(g["n_cases"])):
            p = f"s{k}_"
            temp, top_p, _seed = g[p + "meta"]
            logits, dl = g[p + "logits"], g[p + "draft_logits"]
            n = logits.shape[0]
            par, tok, nr = _aug_batch([g[p + "parent"]], [g[p + "tokens"]], n)
            res = run_virtual_sharded_stochastic(_dev(logits[None], torch.float32), _dev(dl[None], torch.float32),
                                                 float(temp), float(top_p), _dev(par, torch.int32),
                                                 _dev(nr, torch.int32), _dev(tok, torch.int32),
                                                 _dev(g[p + "uniforms"][None], torch.float64), world,
                                                 want_residual=True)
            torch.cuda.synchronize()
            want = (list(g[p + "path"]), int(g[p + "next"]), int(g[p + "used"]))
            for rk, rr in enumerate(res):
                assert int(rr.err[0]) == 0
                plen = int(rr.path_len[0])
                got = (rr.path[0, :plen].cpu().tolist(), int(rr.next_token[0]), int(rr.uniforms_used[0]))
                assert got == want, (world, k, rk, got, want)
            resid = np.concatenate([rr.residual[0].cpu().numpy() for rr in res])
            np.testing.assert_allclose(resid, g[p + "residual"], atol=2e-6)


@pytest.mark.parametrize("world", [2, 8])
def test_sharded_stochastic_full_vocab_vs_oracle(world):
    """128,256-entry vocabulary split over `world` ranks, the 64-row tree,
    T = 1, top-p 0.9, device Philox uniforms: same path / next / used as the
    float64 oracle and as the unsharded kernel."""
    from paper_2508_08192_b200.sampling import accept_stochastic, device_uniforms
    from paper_2508_08192_b200.sharding import run_virtual_sharded_stochastic

    B, V, T, top_p = 3, 128256, 1.0, 0.9
    aug, tl, dl, tokens, seeds, steps = _stochastic_case(B, V, TREE64, T, top_p, seed=23)
    R = len(aug)
    par = torch.tensor([aug] * B, dtype=torch.int32, device="cuda")
    nr = torch.full((B,), R, dtype=torch.int32, device="cuda")
    tl_d, dl_d, tok_d = torch.tensor(tl, device="cuda"), torch.tensor(dl, device="cuda"), torch.tensor(tokens,
                                                                                                         device="cuda")
    uni = device_uniforms(_i64(seeds), _i64(steps), R)
    res = run_virtual_sharded_stochastic(tl_d, dl_d, T, top_p, par, nr, tok_d, uni, world)
    ref = accept_stochastic(tl_d, dl_d, T, top_p, par, nr, tok_d, uni)
    torch.cuda.synchronize()
    for b in range(B):
        path, nxt, _res, used = _oracle_accept(aug, tl[b], dl[b], tokens[b], uni[b].cpu().numpy(), T, top_p)
        for rr in res + [ref]:
            assert int(rr.err[0]) == 0
            plen = int(rr.path_len[b])
            assert rr.path[b, :plen].cpu().tolist() == list(path), b
            assert int(rr.next_token[b]) == nxt and int(rr.uniforms_used[b]) == used, b


def test_sharded_stochastic_nan_flags_every_rank():
    from paper_2508_08192_b200.sharding import run_virtual_sharded_stochastic

    aug = O.augment((-1, -1, 0))
    R, V = len(aug), 300
    rng = np.random.default_rng(1)
    tl = rng.normal(size=(1, R, V)).astype(np.float32)
    tl[0, 1, 250] = np.nan  # lives on the last of 2 ranks
    res = run_virtual_sharded_stochastic(_dev(tl, torch.float32), _dev(tl, torch.float32), 1.0, 0.9,
                                         _dev(np.array([aug]), torch.int32), _dev(np.array([R]), torch.int32),
                                         _dev(np.array([[0, 1, 2, 3]]), torch.int32),
                                         _dev(rng.random((1, R)), torch.float64), 2)
    torch.cuda.synchronize()
    for rr in res:
        assert int(rr.err[0]) & 2
        assert int(rr.path_len[0]) == 0


def _gloo_rank(rank, world, port, case, q):
    import os

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    import torch.distributed as dist

    from paper_2508_08192_b200 import _lib
    from paper_2508_08192_b200.sharding import ShardedStochasticAcceptor, shard_for

    _lib.load()
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        aug, tl, dl, tokens, seeds, steps, T, top_p = case
        B, R, V = tl.shape
        sh = shard_for(rank, world, world, world, V)
        acc = ShardedStochasticAcceptor(sh)
        res = acc(_dev(tl[:, :, sh.v_lo:sh.v_hi], torch.float32), _dev(dl[:, :, sh.v_lo:sh.v_hi], torch.float32), T,
                  top_p, _dev(np.array([aug] * B), torch.int32), _dev(np.full(B, R), torch.int32),
                  _dev(tokens, torch.int32), seeds=_i64(seeds), steps=_i64(steps))
        torch.cuda.synchronize()
        q.put((rank, int(res.err[0]), res.path.cpu().numpy(), res.path_len.cpu().numpy(),
               res.next_token.cpu().numpy(), res.uniforms_used.cpu().numpy()))
    finally:
        dist.destroy_process_group()


def test_sharded_stochastic_two_processes_gloo():
    """The real torch.distributed protocol (two processes sharing cuda:0 over
    gloo; NCCL runs the same calls on a multi-GPU box) vs the oracle."""
    import socket

    import torch.multiprocessing as mp

    B, V, T, top_p = 2, 4099, 0.8, 0.95
    case = _stochastic_case(B, V, TREE64, T, top_p, seed=31) + (T, top_p)
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_gloo_rank, args=(r, 2, port, case, q)) for r in range(2)]
    for p in procs:
        p.start()
    out = [q.get(timeout=300) for _ in procs]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    aug, tl, dl, tokens, seeds, steps = case[:6]
    R = len(aug)
    for rank, err, path, plen, nxt, used in out:
        assert err == 0
        for b in range(B):
            uni = O.rank_sliced_uniforms(seeds[b], steps[b], 1, R)[0]
            want = _oracle_accept(aug, tl[b], dl[b], tokens[b], uni, T, top_p)
            assert list(path[b, :plen[b]]) == list(want[0]) and nxt[b] == want[1] and used[b] == want[3], (rank, b)


@pytest.mark.parametrize("B", [1, 3])
def test_accept_greedy_small_batch_split_rows_vs_oracle(B):
    """bs 1-3 at V = 128,256: each row's vocabulary is scanned by several CTAs
    (partial keys); ties planted across segment boundaries must resolve to
    the lowest index, NaN-free rows bit-exact vs the oracle walk."""
    from paper_2508_08192_b200.sampling import accept_greedy

    V = 128256
    rng = np.random.default_rng(41 + B)
    aug = O.augment(tuple(TREE64))
    R = len(aug)
    lg = (2.0 * rng.normal(size=(B, R, V))).astype(np.float32)
    for b in range(B):
        for r in range(0, R, 3):  # tie of the row max in two far-apart segments
            i, j = sorted(rng.choice(V, size=2, replace=False))
            lg[b, r, i] = lg[b, r, j] = 50.0
    am = lg.argmax(axis=-1)
    tokens = np.zeros((B, R), dtype=np.int32)
    for b in range(B):
        for i in range(1, R):
            tokens[b, i] = am[b, aug[i]] if rng.random() < 0.7 else rng.integers(V)
    res = accept_greedy(torch.tensor(lg, device="cuda"), torch.tensor([aug] * B, dtype=torch.int32, device="cuda"),
                        torch.full((B,), R, dtype=torch.int32, device="cuda"), torch.tensor(tokens, device="cuda"))
    torch.cuda.synchronize()
    for b in range(B):
        path, nxt, used = O.greedy_walk(tuple(p - 1 if p > 0 else -1 for p in aug[1:]), tokens[b, 1:], am[b])
        plen = int(res.path_len[b])
        assert res.path[b, :plen].cpu().tolist() == list(path)
        assert int(res.next_token[b]) == nxt and int(res.uniforms_used[b]) == used


# ---------------------------------------------------------------------------
# FSM-masked rows (guided decoding, target_dist(allowed=...), sampling.py:94-99)
# ---------------------------------------------------------------------------

def _fsm_masks(rng, B, R, V, density):
    m = rng.random((B, R, V)) < density
    m[:, :, 0] = True  # every row keeps at least one token
    return m


def test_accept_greedy_fsm_masked_vs_oracle():
    from paper_2508_08192_b200.sampling import accept_greedy, pack_allowed

    B, V = 3, 5003
    rng = np.random.default_rng(8)
    aug = O.augment(tuple(TREE64))
    R = len(aug)
    lg = (2.0 * rng.normal(size=(B, R, V))).astype(np.float32)
    allowed = _fsm_masks(rng, B, R, V, 0.3)
    masked = np.where(allowed, lg, -np.inf)
    am = masked.argmax(-1)
    tokens = np.zeros((B, R), dtype=np.int32)
    for b in range(B):
        for i in range(1, R):
            tokens[b, i] = am[b, aug[i]] if rng.random() < 0.7 else rng.integers(V)
    res = accept_greedy(torch.tensor(lg, device="cuda"), torch.tensor([aug] * B, dtype=torch.int32, device="cuda"),
                        torch.full((B,), R, dtype=torch.int32, device="cuda"), torch.tensor(tokens, device="cuda"),
                        allowed=pack_allowed(torch.tensor(allowed, device="cuda")))
    torch.cuda.synchronize()
    assert int(res.err[0]) == 0
    for b in range(B):
        # the reference: target_dist(row, 0, 1, allowed) = one-hot at the allowed argmax
        dists = [O.target_dist(lg[b, r].astype(np.float64), 0.0, 1.0, allowed[b, r]) for r in range(R)]
        path, nxt, used = O.greedy_walk(tuple(p - 1 if p > 0 else -1 for p in aug[1:]), tokens[b, 1:],
                                        [int(np.argmax(d)) for d in dists])
        plen = int(res.path_len[b])
        assert res.path[b, :plen].cpu().tolist() == list(path)
        assert int(res.next_token[b]) == nxt and int(res.uniforms_used[b]) == used


@pytest.mark.parametrize("top_p,lazy", [(0.9, True), (0.9, False), (1.0, True)])
def test_accept_stochastic_fsm_masked_vs_oracle(top_p, lazy):
    from paper_2508_08192_b200.sampling import StochasticAcceptor, pack_allowed

    def accept_stochastic(*a, **k):
        return StochasticAcceptor(lazy=lazy)(*a, **k)

    B, V, T = 3, 8192, 1.0
    rng = np.random.default_rng(9)
    aug = O.augment(tuple(TREE64))
    R = len(aug)
    tl = (2.0 * rng.normal(size=(B, R, V))).astype(np.float32)
    dl = (tl + 0.5 * rng.normal(size=(B, R, V))).astype(np.float32)
    allowed = _fsm_masks(rng, B, R, V, 0.4)
    tokens = np.zeros((B, R), dtype=np.int32)
    for b in range(B):
        for i in range(1, R):
            q = O.target_dist(dl[b, aug[i]].astype(np.float64), T, 1.0, allowed[b, aug[i]])
            tokens[b, i] = int(O.sample_from(q, rng.random()))
    seeds, steps = [77 + b for b in range(B)], [6 for _ in range(B)]
    res = accept_stochastic(torch.tensor(tl, device="cuda"), torch.tensor(dl, device="cuda"), T, top_p,
                            torch.tensor([aug] * B, dtype=torch.int32, device="cuda"),
                            torch.full((B,), R, dtype=torch.int32, device="cuda"), torch.tensor(tokens, device="cuda"),
                            seeds=_i64(seeds), steps=_i64(steps),
                            allowed=pack_allowed(torch.tensor(allowed, device="cuda")))
    torch.cuda.synchronize()
    assert int(res.err[0]) == 0
    for b in range(B):
        uni = O.rank_sliced_uniforms(seeds[b], steps[b], 1, R)[0]
        tdists = [O.target_dist(tl[b, r].astype(np.float64), T, top_p, allowed[b, r]) for r in range(R)]
        nd = [O.target_dist(dl[b, aug[i]].astype(np.float64), T, 1.0, allowed[b, aug[i]]) for i in range(1, R)]
        path, nxt, _res, used = O.mss_verify(tuple(p - 1 if p > 0 else -1 for p in aug[1:]), tokens[b, 1:], nd,
                                             tdists, uni)
        plen = int(res.path_len[b])
        assert res.path[b, :plen].cpu().tolist() == list(path), b
        assert int(res.next_token[b]) == nxt and int(res.uniforms_used[b]) == used, b


def test_fsm_dead_row_raises_flag():
    from paper_2508_08192_b200.sampling import accept_greedy, accept_stochastic, pack_allowed

    aug = O.augment((-1, -1, 0))
    R, V = len(aug), 300
    rng = np.random.default_rng(3)
    lg = torch.tensor(rng.normal(size=(1, R, V)).astype(np.float32), device="cuda")
    allowed = np.ones((1, R, V), dtype=bool)
    allowed[0, 1] = False  # dead FSM state on row 1
    words = pack_allowed(torch.tensor(allowed, device="cuda"))
    from paper_2508_08192_b200.sampling import StochasticAcceptor

    par = torch.tensor([aug], dtype=torch.int32, device="cuda")
    nr = torch.tensor([R], dtype=torch.int32, device="cuda")
    tok = torch.zeros((1, R), dtype=torch.int32, device="cuda")
    g = accept_greedy(lg, par, nr, tok, allowed=words)
    s = accept_stochastic(lg, lg, 1.0, 0.9, par, nr, tok, torch.tensor(rng.random((1, R)), device="cuda"),
                          allowed=words)
    # lazy: the dead row is never visited (path stops at the root); the
    # validation scan still raises, like the reference's every-row target_dist
    s2 = StochasticAcceptor(lazy=True)(lg, lg, 1.0, 0.9, par, nr, tok,
                                       torch.tensor(rng.random((1, R)), device="cuda"), allowed=words)
    torch.cuda.synchronize()
    assert int(g.err[0]) & 32 and int(s.err[0]) & 32 and int(s2.err[0]) & 32


@pytest.mark.parametrize("scan_sms", [None, "0"])
@pytest.mark.parametrize("V", [4096, 4099])
def test_lazy_validation_scan_error_semantics(V, scan_sms, monkeypatch):
    """The lazy walk reduces only the rows it visits; the validation scan
    (persistent on 52 of 148 SMs by default, SDB_VALIDATE_SMS=0: one-row
    CTAs) must still raise exactly where the reference does: target_dist of
    EVERY tree row and the draft q of every PARENT row (engine.py:474-475,
    numcore.py:47-48) -- a NaN in a draft leaf row or past a sequence's
    n_rows is never read by the reference and must not raise."""
    from paper_2508_08192_b200.sampling import StochasticAcceptor, tree_levels

    if scan_sms is not None:
        monkeypatch.setenv("SDB_VALIDATE_SMS", scan_sms)
    B, T, top_p = 24, 1.0, 0.9
    aug, tl, dl, tokens, seeds, steps = _stochastic_case(B, V, TREE64, T, top_p, seed=77)
    R = len(aug)
    n_rows = np.full((B,), R, dtype=np.int32)
    n_rows[5] = R - 7  # ragged: rows >= R - 7 of sequence 5 are not part of its tree
    parents = set(p for p in aug if p >= 0)
    leaf = max(r for r in range(R) if r not in parents)
    par_row = max(parents)
    par = torch.tensor([aug] * B, dtype=torch.int32, device="cuda")
    acc = StochasticAcceptor(lazy=True, levels=tree_levels(par))

    def run(t, d):
        res = acc(torch.tensor(t, device="cuda"), torch.tensor(d, device="cuda"), T, top_p, par,
                  torch.tensor(n_rows, device="cuda"), torch.tensor(tokens, device="cuda"), seeds=_i64(seeds),
                  steps=_i64(steps))
        torch.cuda.synchronize()
        return int(res.err[0])

    assert run(tl, dl) == 0
    cases = [
        ("target, last row of the last sequence", True, B - 1, R - 1, True),
        ("target, unvisited middle row", True, 13, R // 2, True),
        ("draft, a parent row", False, 7, par_row, True),
        ("draft, a leaf row", False, 7, leaf, False),
        ("target, past n_rows", True, 5, R - 2, False),
    ]
    for what, target, b, r, raises in cases:
        t, d = tl.copy(), dl.copy()
        (t if target else d)[b, r, V // 3] = np.nan
        err = run(t, d)
        assert bool(err & 2) == raises, what
