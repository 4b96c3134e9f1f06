"""Parity of the exact configurations bench.py times.

Every number the bench reports has a matching oracle check here, on the
bench's own inputs (``bench.make_inputs``) and through the same call path:

* C3 (70B shapes, bs 32, ctx 8192, 64-row tree): ``TreeVerifier`` as the
  bench builds it -- the auto SM reserve (attention on 64 CTA pairs) with the
  greedy scan running concurrently on a forked graph branch -- captured into
  a CUDA graph and replayed.  All 32 accepted paths / bonus tokens / uniform
  counts are compared with the oracle's argmax walk, and out / LSE of sampled
  (sequence, KV head) slices with the float64 oracle (attention.py:131-151).
* C4 (405B shapes: 128q / 8kv, g = 16, bs 64, ctx 32768): the same, with the
  greedy scan fused into the CTA-pair attention kernel (the bench's plan).
* C5 (stochastic top-p acceptance, bs 64, V = 128,256): lazy and eager modes
  vs target_dist + mss_verify (sampling.py:87-202) on every sequence.
* Vocab-sharded greedy acceptance (ShardedGreedyAcceptor) over two real
  processes (gloo, sharing cuda:0): vocab_offset != 0, ties across the shard
  boundary, a NaN on one rank raising on both.

Needs a B200."""

import os
import socket

import numpy as np
import pytest

torch = pytest.importorskip("torch")

pytestmark = pytest.mark.gpu

import bench  # noqa: E402
from oracle import specdec_oracle as O  # noqa: E402


@pytest.fixture(scope="module", autouse=True)
def _lib_loaded():
    from paper_2508_08192_b200 import _lib

    _lib.load()
    bench.TREE = bench.TREE64


def _f64(t):
    return t.float().cpu().numpy().astype(np.float64)


def _slice_oracle(x, b, kvh, g, aug, scale):
    """Float64 oracle of one (sequence, KV head): out [R, g, d], lse [g, R].
    Only the sequence's own pages are gathered to the host."""
    c = int(x.ctx_len[b])
    bs = x.k_pool.shape[2]
    n_pages = -(-c // bs)
    pages = x.block_table[b, :n_pages].long()
    kp = _f64(x.k_pool[pages][:, kvh:kvh + 1])
    vp = _f64(x.v_pool[pages][:, kvh:kvh + 1])
    q = _f64(x.q[b:b + 1, :, kvh * g:(kvh + 1) * g])
    tk = _f64(x.tree_k[b:b + 1, :, kvh:kvh + 1])
    tv = _f64(x.tree_v[b:b + 1, :, kvh:kvh + 1])
    out, lse = O.tree_verify_attention_batch(q, kp, vp, np.arange(n_pages)[None], np.array([c]), tk, tv, [aug],
                                             scale)
    return out[0], lse[0]


def _check_greedy_paths(x, acc, raw_parent):
    logits = x.logits.cpu().numpy()
    tokens = x.tokens.cpu().numpy()
    path = acc.path.cpu().numpy()
    plen = acc.path_len.cpu().numpy()
    nxt = acc.next_token.cpu().numpy()
    used = acc.uniforms_used.cpu().numpy()
    for b in range(logits.shape[0]):
        want_path, want_next, want_used = O.greedy_walk(raw_parent, tokens[b, 1:], np.argmax(logits[b], axis=-1))
        assert list(path[b, :plen[b]]) == want_path, b
        assert int(nxt[b]) == want_next and int(used[b]) == want_used, b
    return float(plen.mean())


def _run_bench_step(config, mode="greedy", tree="64"):
    from paper_2508_08192_b200.sharding import shard_for
    from paper_2508_08192_b200.verify import TreeVerifier

    bench.TREE = bench.TREES[tree]
    cfg = bench.CONFIGS[config]
    dev = torch.device("cuda", 0)
    shard = shard_for(0, 1, cfg["Hq"], cfg["Hkv"], cfg["V"])
    x, R = bench.make_inputs(cfg, shard, dev, mode=mode)
    aug = tuple(bench._augment(bench.TREE))
    ver = TreeVerifier(scale=cfg["d"] ** -0.5, temperature=0.0, max_ctx=cfg["ctx"],
                       tree_levels=bench._tree_levels(aug))
    ver.capture(x)
    for _ in range(3):
        out, lse, acc, terr = ver.replay()
    torch.cuda.synchronize()
    assert int(terr.abs().sum()) == 0
    acc.raise_if_error()
    return cfg, x, R, aug, out, lse, acc


def _check_slices(cfg, x, aug, out, lse, slices):
    g = cfg["Hq"] // cfg["Hkv"]
    scale = cfg["d"] ** -0.5
    for b, kvh in slices:
        want_o, want_l = _slice_oracle(x, b, kvh, g, aug, scale)
        got_o = out[b, :, kvh * g:(kvh + 1) * g].float().cpu().numpy()
        got_l = lse[b, kvh * g:(kvh + 1) * g].cpu().numpy()
        err = np.abs(got_o - want_o)
        assert err.max() < 2e-2 and err.mean() < 2e-3, (b, kvh, err.max(), err.mean())
        assert np.abs(got_l - want_l).max() < 2e-3, (b, kvh)


def test_c3_bench_step_vs_oracle():
    """C3 exactly as bench.py times it: reserve plan + concurrent greedy scan,
    graph-replayed; all 32 paths and three (sequence, KV head) slices."""
    from paper_2508_08192_b200.verify import TreeVerifier, _num_sms

    cfg, x, R, aug, out, lse, acc = _run_bench_step("c3")
    ver = TreeVerifier(scale=cfg["d"] ** -0.5, max_ctx=cfg["ctx"])
    # the plan under test: SMs left to the concurrent acceptance
    assert ver._auto_reserve(x, cfg["B"], R, _num_sms(x.q.device)) >= 8
    _check_greedy_paths(x, acc, tuple(bench.TREE))
    _check_slices(cfg, x, aug, out, lse, [(0, 0), (13, 5), (31, 7)])


@pytest.mark.parametrize("tree", ["chain3", "n8", "65"])
def test_c3_other_trees_bench_step_vs_oracle(tree):
    """The bench's other C3 trees: the HBM-bound contrast trees chain-3
    (R = 4, R*g = 32 rows per KV head: one part-filled 128-row MMA tile) and
    N8 (R = 9, R*g = 72), and the R = 65 variant (520 rows per KV head)."""
    try:
        cfg, x, R, aug, out, lse, acc = _run_bench_step("c3", tree=tree)
        _check_greedy_paths(x, acc, tuple(bench.TREE))
        _check_slices(cfg, x, aug, out, lse, [(0, 0), (17, 6), (31, 7)])
    finally:
        bench.TREE = bench.TREE64


def test_c4_bench_step_vs_oracle():
    """C4 (405B shapes, g = 16: a Q TMA box {64, 16, 1, 8} and four 256-row
    pair tiles per KV head; ctx 32768 = 256 prefix tiles per unit) with the
    greedy scan fused into the attention kernel, as the bench runs it."""
    from paper_2508_08192_b200.verify import TreeVerifier

    cfg, x, R, aug, out, lse, acc = _run_bench_step("c4")
    ver = TreeVerifier(scale=cfg["d"] ** -0.5, max_ctx=cfg["ctx"])
    assert ver._scan_hides(x, cfg["B"], R, x.q.device)  # the fused-scan plan is the one under test
    _check_greedy_paths(x, acc, tuple(bench.TREE))
    _check_slices(cfg, x, aug, out, lse, [(0, 0), (37, 3), (63, 7)])


@pytest.mark.parametrize("lazy", [True, False])
def test_c5_stochastic_all_sequences_vs_oracle(lazy):
    """C5 inputs (bs 64, 64-row tree, V = 128,256, T 1, top-p 0.9, device
    Philox uniforms): lazy walk (8-CTA clusters in two waves + the
    concurrent validation scan) and eager row stats, every sequence exact."""
    from paper_2508_08192_b200.sampling import StochasticAcceptor
    from paper_2508_08192_b200.sharding import shard_for

    cfg = bench.CONFIGS["c5"]
    dev = torch.device("cuda", 0)
    x, R = bench.make_inputs(cfg, shard_for(0, 1, cfg["Hq"], cfg["Hkv"], cfg["V"]), dev, mode="stochastic")
    aug = tuple(bench._augment(bench.TREE))
    acc = StochasticAcceptor(lazy=lazy, levels=bench._tree_levels(aug))
    res = acc(x.logits, x.draft_logits, bench.TEMPERATURE, bench.TOP_P, x.parent, x.n_rows, x.tokens,
              seeds=x.seeds, steps=x.steps)
    torch.cuda.synchronize()
    res.raise_if_error()
    raw = tuple(bench.TREE)
    tokens = x.tokens.cpu().numpy()
    seeds, steps = x.seeds.cpu().numpy(), x.steps.cpu().numpy()
    path, plen = res.path.cpu().numpy(), res.path_len.cpu().numpy()
    nxt, used = res.next_token.cpu().numpy(), res.uniforms_used.cpu().numpy()
    for b in range(cfg["B"]):
        def tdist(i, b=b):
            return O.target_dist(x.logits[b, i].double().cpu().numpy(), bench.TEMPERATURE, bench.TOP_P)

        qmemo = {}

        def qdist(c, b=b):
            row = aug[1 + c]  # the draft q of the node's parent row (engine.py:405-407)
            if row not in qmemo:
                qmemo[row] = O.target_dist(x.draft_logits[b, row].double().cpu().numpy(), bench.TEMPERATURE, 1.0)
            return qmemo[row]

        uni = O.rank_sliced_uniforms(int(seeds[b]), int(steps[b]), 1, R)[0]
        want_path, want_next, _resid, want_used = O.mss_verify(raw, tokens[b, 1:], qdist, tdist, uni)
        assert list(path[b, :plen[b]]) == want_path, b
        assert int(nxt[b]) == want_next and int(used[b]) == want_used, b


# ---------------------------------------------------------------------------
# vocab-sharded greedy acceptance over two processes
# ---------------------------------------------------------------------------

def _greedy_case(B, V, seed):
    rng = np.random.default_rng(seed)
    aug = O.augment(tuple(bench.TREE64))
    R = len(aug)
    tl = (2.0 * rng.normal(size=(B, R, V))).astype(np.float32)
    lo1 = V // 2 + V % 2  # rank 1's first column at world 2 (shard_for)
    tl[0, 0, lo1 - 1] = tl[0, 0, lo1] = 50.0   # tie across the shard boundary -> rank 0's index
    tl[1, 0, lo1] = tl[1, 0, V - 1] = 50.0     # tie inside rank 1 -> its lowest index
    tl[2, 0, 7] = tl[2, 0, lo1 + 5] = 50.0     # tie across ranks, far apart
    tl[3, :, :] = np.round(tl[3])              # integer logits: many ties in every row
    am = np.argmax(tl, axis=-1)
    tokens = np.zeros((B, R), dtype=np.int32)
    for b in range(B):
        for i in range(1, R):
            tokens[b, i] = am[b, aug[i]] if rng.random() < 0.7 else rng.integers(V)
    return aug, tl, tokens


def _greedy_rank(rank, world, port, case, nan_case, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    import torch.distributed as dist

    from paper_2508_08192_b200 import _lib
    from paper_2508_08192_b200.sharding import ShardedGreedyAcceptor, shard_for

    _lib.load()
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        out = []
        for aug, tl, tokens in (case, nan_case):
            B, R, V = tl.shape
            sh = shard_for(rank, world, world, world, V)
            res = ShardedGreedyAcceptor(sh)(torch.tensor(tl[:, :, sh.v_lo:sh.v_hi], device="cuda"),
                                            torch.tensor(np.array([aug] * B), dtype=torch.int32, device="cuda"),
                                            torch.full((B,), R, dtype=torch.int32, device="cuda"),
                                            torch.tensor(tokens, device="cuda"))
            torch.cuda.synchronize()
            out.append((int(res.err[0]), res.path.cpu().numpy(), res.path_len.cpu().numpy(),
                        res.next_token.cpu().numpy(), res.uniforms_used.cpu().numpy(), sh.v_lo))
        q.put((rank, out))
    finally:
        dist.destroy_process_group()


def test_sharded_greedy_two_processes_gloo():
    """ShardedGreedyAcceptor on two processes: sdb_argmax_keys with
    vocab_offset != 0 on rank 1, one all-reduce(MAX) of the packed keys and
    the error word, the same walk on both ranks == the oracle's argmax walk
    (numpy lowest-index ties, numcore.py:51-55).  A NaN that only rank 1
    sees raises on both ranks (softmax_lse, numcore.py:47-48)."""
    import torch.multiprocessing as mp

    B, V = 4, 4099  # odd: rank 0 owns 2050 columns, rank 1 2049 (scalar tails)
    case = _greedy_case(B, V, seed=5)
    aug, tl, tokens = case
    nan_tl = tl.copy()
    nan_tl[2, 9, V - 3] = np.nan  # rank 1's shard only
    nan_case = (aug, nan_tl, tokens)
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_greedy_rank, args=(r, 2, port, case, nan_case, q)) for r in range(2)]
    for p in procs:
        p.start()
    got = dict(q.get(timeout=300) for _ in procs)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert got[1][0][5] > 0  # rank 1's shard starts past 0
    raw = tuple(bench.TREE64)
    for rank in (0, 1):
        err, path, plen, nxt, used, _ = got[rank][0]
        assert err == 0
        for b in range(B):
            want_path, want_next, want_used = O.greedy_walk(raw, tokens[b, 1:], np.argmax(tl[b], axis=-1))
            assert list(path[b, :plen[b]]) == want_path, (rank, b)
            assert int(nxt[b]) == want_next and int(used[b]) == want_used, (rank, b)
        nan_err = got[rank][1][0]
        assert nan_err & 2, rank  # SDB_ERR_NAN on both ranks


@pytest.mark.parametrize("tree", ["64", "chain3"])
def test_context_past_max_ctx_raises_cache_error(tree):
    """A ctx_len beyond the planned max_ctx (the tcgen05 plan covers
    ceil(max_ctx / 128) prefix tiles) raises CacheError through
    TreeVerifier.check() instead of silently dropping keys -- the pair kernel
    (64-row tree) and the 1-CTA kernel (chain-3); within the plan it passes."""
    from paper_2508_08192_b200.kvstore import CacheError
    from paper_2508_08192_b200.sharding import shard_for
    from paper_2508_08192_b200.verify import TreeVerifier

    bench.TREE = bench.TREES[tree]
    cfg = dict(bench.CONFIGS["c3"], B=2, ctx=1024, V=2048)
    x, R = bench.make_inputs(cfg, shard_for(0, 1, cfg["Hq"], cfg["Hkv"], cfg["V"]), torch.device("cuda", 0))
    ok = TreeVerifier(scale=cfg["d"] ** -0.5, max_ctx=1024, kernel=1)
    out, lse, acc, terr = ok.step(x)
    torch.cuda.synchronize()
    ok.check(acc=acc)  # within the plan: no error
    short = TreeVerifier(scale=cfg["d"] ** -0.5, max_ctx=512, kernel=1)
    out, lse, acc, terr = short.step(x)
    torch.cuda.synchronize()
    with pytest.raises(CacheError):
        short.check()
    short.check()  # the word is reset once reported
