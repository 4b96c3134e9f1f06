"""CPU, world_size 2 over gloo: the multi-GPU host protocol of
paper_2508_08192_b200.sharding -- KV-head / vocab partition and the vocab-
sharded greedy acceptance (packed argmax keys + one all-reduce MAX) -- gives
the same argmax / walk as the unsharded reference semantics on every rank."""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from oracle import specdec_oracle as O
from paper_2508_08192_b200.sharding import combine_argmax_keys, key_to_index, shard_for


def _pack_keys(logits, v_lo):
    """Host model of sdb_argmax_keys' key format (sdb_common.cuh argmax_key):
    int64 = int32(orderable(max) ^ 0x80000000) << 32 | (0xFFFFFFFF - index)."""
    rows, v = logits.shape
    keys = np.empty(rows, dtype=np.int64)
    for r in range(rows):
        row = logits[r].astype(np.float32)
        row = np.where(row == 0.0, np.float32(0.0), row)
        bits = row.view(np.uint32).astype(np.uint64)
        neg = (bits & 0x80000000) != 0
        ordv = np.where(neg, (~bits) & 0xFFFFFFFF, bits | 0x80000000)
        best = None
        for j in range(v):
            hi = int(ordv[j]) ^ 0x80000000
            hi = hi - (1 << 32) if hi >= (1 << 31) else hi
            k = (hi << 32) | (0xFFFFFFFF - (v_lo + j))
            if best is None or k > best:
                best = k
        keys[r] = best
    return keys


def test_shard_partition_covers_everything():
    for world in (1, 2, 4, 8):
        shards = [shard_for(r, world, 64, 8, 128256) for r in range(world)]
        assert [s.kv_lo for s in shards] == [r * 8 // world for r in range(world)]
        assert sum(s.n_kv for s in shards) == 8 and sum(s.n_q for s in shards) == 64
        assert shards[0].v_lo == 0 and shards[-1].v_hi == 128256
        for a, b in zip(shards, shards[1:]):
            assert a.v_hi == b.v_lo and a.q_hi == b.q_lo
    with pytest.raises(ValueError):
        shard_for(0, 3, 64, 8, 1000)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        rng = np.random.default_rng(0)
        V = 203  # uneven split across ranks
        parent = O.augment((-1, -1, 0, 0, 1, 2, 2, 5))
        R = len(parent)
        logits = rng.integers(-3, 4, size=(R, V)).astype(np.float32)  # ties everywhere
        logits[2, [10, 150]] = 9.0  # a tie that straddles the shard boundary
        logits[3, 7] = -0.0
        sh = shard_for(rank, world, 8, 2, V)
        local = _pack_keys(logits[:, sh.v_lo:sh.v_hi], sh.v_lo)
        keys = torch.from_numpy(local)
        combine_argmax_keys(keys)
        got = key_to_index(keys).numpy()
        want = np.argmax(logits.astype(np.float64), axis=1)
        tokens = np.array([0] + [int(want[p]) if i % 3 else (int(want[p]) + 1) % V
                                 for i, p in enumerate(parent[1:], 1)])
        path, nxt, used = O.greedy_walk(tuple(p - 1 if p > 0 else -1 for p in parent[1:]), tokens[1:], got)
        q.put((rank, got.tolist(), want.tolist(), path, nxt, used))
    finally:
        dist.destroy_process_group()


def test_vocab_sharded_greedy_acceptance_gloo_world2():
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=120) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    res.sort()
    for rank, got, want, path, nxt, used in res:
        assert got == want, (rank, got, want)
    # every rank walks to the same result without a broadcast
    assert len({(tuple(r[3]), r[4], r[5]) for r in res}) == 1


# ---------------------------------------------------------------------------
# vocab-sharded stochastic acceptance: the phase/collective decomposition of
# csrc/accept_sharded.cu, restated in numpy (oracle/sharded_accept.py), run
# over real gloo collectives on CPU -- every rank must reproduce the unsharded
# reference acceptance (target_dist + mss_verify).
# ---------------------------------------------------------------------------

class _GlooNumpyComm:
    def __init__(self, rank, world):
        self.rank, self.world = rank, world

    def all_gather(self, a):
        t = torch.from_numpy(np.ascontiguousarray(a))
        out = [torch.empty_like(t) for _ in range(self.world)]
        dist.all_gather(out, t)
        return np.stack([o.numpy() for o in out])

    def all_reduce_sum(self, a):
        t = torch.from_numpy(np.ascontiguousarray(a))
        dist.all_reduce(t)
        return t.numpy()

    def all_reduce_max(self, a):
        t = torch.from_numpy(np.ascontiguousarray(a))
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return t.numpy()


def _stoch_cases():
    rng = np.random.default_rng(12)
    cases = []
    trees = [(-1, -1, 0, 0, 1, 2, 2, 5), (-1, 0, 1, 2), (-1, -1, -1, 0, 0, 0, 3)]
    for ci in range(9):
        parent = O.augment(trees[ci % 3])
        R, V = len(parent), (203, 1000, 64)[ci % 3]
        T, top_p = ((1.0, 0.9), (0.7, 0.95), (1.3, 1.0))[ci % 3]
        if ci >= 6:  # integer logits: ties everywhere, also across the shard boundary
            tl = rng.integers(-3, 4, size=(R, V)).astype(np.float32)
            dl = np.where(rng.random((R, V)) < 0.7, tl, rng.integers(-3, 4, size=(R, V))).astype(np.float32)
        else:
            tl = (2.0 * rng.normal(size=(R, V))).astype(np.float32)
            dl = (tl + 0.5 * rng.normal(size=(R, V))).astype(np.float32)
        tokens = np.zeros(R, dtype=np.int64)
        for i in range(1, R):
            q = O.target_dist(dl[parent[i]].astype(np.float64), T, 1.0)
            tokens[i] = O.sample_from(q, rng.random())
        uni = O.rank_sliced_uniforms(77 + ci, 2 * ci + 2, 1, R)[0]
        cases.append((parent, tl, dl, tokens, uni, T, top_p))
    return cases


def _want(case):
    parent, tl, dl, tokens, uni, T, top_p = case
    R = len(parent)
    tdists = [O.target_dist(tl[r].astype(np.float64), T, top_p) for r in range(R)]
    nd = [O.target_dist(dl[parent[i]].astype(np.float64), T, 1.0) for i in range(1, R)]
    path, tok, _res, used = O.mss_verify(tuple(p - 1 if p > 0 else -1 for p in parent[1:]), tokens[1:], nd, tdists,
                                         uni)
    return list(path), int(tok), int(used)


def _stoch_worker(rank, world, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from oracle.sharded_accept import sharded_accept

        comm = _GlooNumpyComm(rank, world)
        res = []
        for parent, tl, dl, tokens, uni, T, top_p in _stoch_cases():
            sh = shard_for(rank, world, world, world, tl.shape[1])
            res.append(sharded_accept(comm, tl[:, sh.v_lo:sh.v_hi], dl[:, sh.v_lo:sh.v_hi], sh.v_lo, tl.shape[1],
                                      parent, tokens, uni, T, top_p))
        q.put((rank, res))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_vocab_sharded_stochastic_protocol_gloo(world):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_stoch_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=300) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    want = [_want(c) for c in _stoch_cases()]
    for rank, got in res:
        for ci, (g, w) in enumerate(zip(got, want)):
            assert (list(g[0]), g[1], g[2]) == w, (world, rank, ci, g, w)
