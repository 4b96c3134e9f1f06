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
    return Shard(rank, world, kv_lo, kv_lo + per, kv_lo * g, (kv_lo + per) * g, v_lo, v_hi)


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
        from .sampling import argmax_keys, greedy_walk

        b, r, v = logits_shard.shape
        keys, err = argmax_keys(logits_shard.reshape(b * r, v), vocab_offset=self.shard.v_lo, stream=stream)
        combine_argmax_keys(keys, self.group)
        res = greedy_walk(keys.reshape(b, r), parent, n_rows, tokens, stream=stream)
        res.err = err
        return res
