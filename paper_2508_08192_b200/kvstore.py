"""Paged KV cache with device-resident pools and the K7 write-back kernel.

``PagedKvCache`` keeps the reference's interface and block discipline
(kvstore.py:113-258: per-sequence block tables drawn from a shared free list,
``alloc_for_step`` tree padding, ``write``/``gather``/``rewind``/``set_len``,
``compact_accepted``) while the pools live in HBM with the layout
``[n_layers][num_blocks][n_kv_heads][block_size][head_dim]`` -- one contiguous
(page, head) slab, which is what the tree-verify attention kernel streams.
The reference's token-major pool is the special case n_kv_heads = 1,
head_dim = dim; ``write``/``gather`` take and return the reference's
``(rows, n_kv_heads * head_dim)`` row matrices either way.

Persistent LRU storage and prefix reuse (kvstore.py:29-110, 261-309) serve
prefill/TTFT, not verification, and are out of scope (SURVEY.md section 2.1
row 5); ``release`` frees the blocks.

``compact_kv`` is the batched device write-back of the accepted path for all
layers and sequences in one launch (engine.py:504-523).
"""

from __future__ import annotations

import numpy as np

from . import _lib


class CacheError(RuntimeError):
    pass


class _SeqState:
    __slots__ = ("table", "length", "written")

    def __init__(self):
        self.table = []
        self.length = 0
        self.written = 0


_ELEM = {"float64": 8, "float32": 4, "bfloat16": 2}


class PagedKvCache:
    def __init__(self, n_layers, dim, n_blocks, block_size=16, store=None, n_kv_heads=1, dtype=None,
                 device="cuda"):
        import torch

        if min(n_layers, dim, n_blocks, block_size) < 1:
            raise CacheError("all cache dimensions must be >= 1")
        if store is not None:
            raise CacheError("persistent KV store (prefix reuse) is out of scope for the verify path")
        if dim % n_kv_heads:
            raise CacheError("dim must be divisible by n_kv_heads")
        self.n_layers = n_layers
        self.dim = dim
        self.n_blocks = n_blocks
        self.block_size = block_size
        self.n_kv_heads = n_kv_heads
        self.head_dim = dim // n_kv_heads
        self.store = None
        self.dtype = dtype if dtype is not None else torch.float64
        shape = (n_layers, n_blocks, n_kv_heads, block_size, self.head_dim)
        # zero-initialised: the attention kernel may read (and mask) rows past
        # the committed length inside the last page; they must be finite.
        self.k_pool = torch.zeros(shape, dtype=self.dtype, device=device)
        self.v_pool = torch.zeros(shape, dtype=self.dtype, device=device)
        self._elem = self.k_pool.element_size()
        self._free = list(range(n_blocks))[::-1]
        self._seqs = {}
        self.stats = {"reused_blocks": 0, "evicted_blocks": 0, "dropped_blocks": 0, "allocated_blocks": 0}

    # -- sequence lifecycle (kvstore.py:130-170) --------------------------
    def new_seq(self, seq):
        if seq in self._seqs:
            raise CacheError(f"sequence {seq!r} already exists")
        self._seqs[seq] = _SeqState()

    def _state(self, seq):
        try:
            return self._seqs[seq]
        except KeyError:
            raise CacheError(f"unknown sequence {seq!r}") from None

    def committed_len(self, seq):
        return self._state(seq).length

    def written_len(self, seq):
        return self._state(seq).written

    def set_len(self, seq, n):
        if n < 0:
            raise CacheError("length must be >= 0")
        self._state(seq).length = n

    def release(self, seq, keys=()):
        st = self._state(seq)
        self._free.extend(st.table)
        del self._seqs[seq]

    @property
    def free_blocks(self):
        return len(self._free)

    @property
    def occupancy(self):
        return self.n_blocks - len(self._free)

    # -- allocation (kvstore.py:185-203) ----------------------------------
    def _grab_block(self):
        if not self._free:
            raise CacheError("block pool exhausted")
        self.stats["allocated_blocks"] += 1
        return self._free.pop()

    def ensure(self, seq, n_positions):
        st = self._state(seq)
        while len(st.table) * self.block_size < n_positions:
            st.table.append(self._grab_block())

    def alloc_for_step(self, seq, n_draft_nodes):
        """Committed length + draft nodes + bonus (kvstore.py:200-203)."""
        self.ensure(seq, self._state(seq).length + n_draft_nodes + 1)

    def block_table(self, seq):
        return list(self._state(seq).table)

    def block_table_tensor(self, seqs, max_blocks=None):
        import torch

        tabs = [self._state(s).table for s in seqs]
        mb = max_blocks or max(1, max(len(t) for t in tabs))
        out = np.zeros((len(tabs), mb), dtype=np.int32)
        for i, t in enumerate(tabs):
            out[i, :len(t)] = t
        return torch.from_numpy(out).to(self.k_pool.device)

    # -- data movement (kvstore.py:217-258) -------------------------------
    def _rows_tensor(self, rows):
        import torch

        if isinstance(rows, torch.Tensor):
            t = rows.to(device=self.k_pool.device, dtype=self.dtype)
        else:
            t = torch.as_tensor(np.asarray(rows), dtype=self.dtype, device=self.k_pool.device)
        return t.reshape(t.shape[0], self.dim).contiguous()

    def write(self, seq, layer, start, k_rows, v_rows):
        st = self._state(seq)
        n = k_rows.shape[0]
        if start + n > len(st.table) * self.block_size:
            raise CacheError("write past allocated blocks")
        if n:
            table = self.block_table_tensor([seq])[0]
            for pool, rows in ((self.k_pool, k_rows), (self.v_pool, v_rows)):
                t = self._rows_tensor(rows)
                rc = _lib.lib().sdb_paged_write(_lib.ptr(pool[layer]), _lib.ptr(table), int(start), _lib.ptr(t), n,
                                                self.n_kv_heads, self.head_dim, self.block_size, self._elem,
                                                _lib.stream_ptr())
                _lib.check(rc, "paged_write")
        st.written = max(st.written, start + n)

    def write_all(self, seq, start, k_by_layer, v_by_layer):
        for layer in range(self.n_layers):
            self.write(seq, layer, start, k_by_layer[layer], v_by_layer[layer])

    def compact_accepted(self, seq, start, k_by_layer, v_by_layer):
        self.write_all(seq, start, k_by_layer, v_by_layer)

    def gather_device(self, seq, layer, n):
        """Rows [0, n) of one layer as device tensors (n, dim)."""
        import torch

        st = self._state(seq)
        if n > st.written:
            raise CacheError(f"gather {n} rows but only {st.written} written")
        out = []
        table = self.block_table_tensor([seq])[0]
        for pool in (self.k_pool, self.v_pool):
            t = torch.empty((n, self.dim), dtype=self.dtype, device=pool.device)
            if n:
                rc = _lib.lib().sdb_paged_gather(_lib.ptr(pool[layer]), _lib.ptr(table), 0, _lib.ptr(t), n,
                                                 self.n_kv_heads, self.head_dim, self.block_size, self._elem,
                                                 _lib.stream_ptr())
                _lib.check(rc, "paged_gather")
            out.append(t)
        return out[0], out[1]

    def gather(self, seq, layer, n):
        k, v = self.gather_device(seq, layer, n)
        if k.dtype == __import__("torch").bfloat16:
            k, v = k.float(), v.float()
        return k.cpu().numpy(), v.cpu().numpy()

    def rewind(self, seq, new_len):
        st = self._state(seq)
        if new_len > st.written:
            raise CacheError("rewind past written length")
        keep = -(-new_len // self.block_size)
        self._free.extend(st.table[keep:])
        del st.table[keep:]
        st.written = new_len
        st.length = new_len


# ---------------------------------------------------------------------------
# batched device write-back
# ---------------------------------------------------------------------------

def compact_kv(tree_k, tree_v, k_pools, v_pools, block_table, ctx_len, path, path_len, n_keep=None, stream=None,
               err=None):
    """Write rows [0] + [1 + a for a in path[:n_keep-1]] of every sequence's
    tree K/V into its pages at positions ctx_len.. for every layer.
    Positions past a sequence's mapped blocks are not written; they set
    SDB_ERR_CACHE in ``err`` (int32 [1], e.g. the acceptance's error word).

    tree_k/v [L, B, R, Hkv, d]; k_pools/v_pools [L, num_blocks, Hkv, bs, d];
    block_table int32 [B, max_blocks]; ctx_len / path_len / n_keep int32 [B];
    path int32 [B, R] (draft-node indices).  One launch, no host sync."""
    n_layers, b, r, hkv, d = tree_k.shape
    bs = k_pools.shape[3]
    if k_pools.shape[2] != hkv or k_pools.shape[4] != d or k_pools.dtype != tree_k.dtype:
        raise CacheError("compact_kv: pool / tree shape mismatch")
    layer_stride = k_pools.stride(0)
    rc = _lib.lib().sdb_compact_kv(_lib.ptr(tree_k), _lib.ptr(tree_v), _lib.ptr(k_pools), _lib.ptr(v_pools),
                                   layer_stride, _lib.ptr(block_table), block_table.shape[1], _lib.ptr(ctx_len),
                                   _lib.ptr(path), _lib.ptr(path_len), _lib.ptr(n_keep), n_layers, b, r, hkv, d, bs,
                                   tree_k.element_size(), _lib.ptr(err), _lib.stream_ptr(stream))
    _lib.check(rc, "compact_kv")


# ---------------------------------------------------------------------------
# bookkeeping either side of the step
# ---------------------------------------------------------------------------

def compact_draft_kv(suffix_k, suffix_v, k_pools, v_pools, block_table, ctx_len, path, path_len, n_keep=None,
                     stream=None, err=None):
    """Draft-cache write-back (engine.py:524-531): rows path[:n_keep-1] of the
    draft's carried suffix K/V [L, B, n_src, Hkv, d] (realized draft nodes, no
    root row) into the draft pages at positions ctx_len + 1 .. (= L)."""
    n_layers, b, n_src, hkv, d = suffix_k.shape
    bs = k_pools.shape[3]
    if k_pools.shape[2] != hkv or k_pools.shape[4] != d or k_pools.dtype != suffix_k.dtype:
        raise CacheError("compact_draft_kv: pool / suffix shape mismatch")
    rc = _lib.lib().sdb_compact_draft_kv(_lib.ptr(suffix_k), _lib.ptr(suffix_v), _lib.ptr(k_pools),
                                         _lib.ptr(v_pools), k_pools.stride(0), _lib.ptr(block_table),
                                         block_table.shape[1], _lib.ptr(ctx_len), _lib.ptr(path), _lib.ptr(path_len),
                                         _lib.ptr(n_keep), n_layers, b, path.shape[1], n_src, hkv, d, bs,
                                         suffix_k.element_size(), _lib.ptr(err), _lib.stream_ptr(stream))
    _lib.check(rc, "compact_draft_kv")


def tape_append(hidden, tape, tape_len, path, path_len, err, n_keep=None, stream=None):
    """HiddenTape.append_rows of the kept rows (engine.py:532-533): rows [0] +
    [1 + a for a in path[:n_keep-1]] of hidden [B, R, dim] appended to tape
    [B, cap, dim] at tape_len [B] (advanced in place)."""
    b, r, dim = hidden.shape
    if tape.shape[0] != b or tape.shape[2] != dim or tape.dtype != hidden.dtype:
        raise CacheError("tape_append: tape / hidden shape mismatch")
    rc = _lib.lib().sdb_tape_append(_lib.ptr(hidden), _lib.ptr(tape), tape.shape[1], _lib.ptr(tape_len),
                                    _lib.ptr(path), _lib.ptr(path_len), _lib.ptr(n_keep), b, r,
                                    dim * hidden.element_size(), _lib.ptr(err), _lib.stream_ptr(stream))
    _lib.check(rc, "tape_append")


class DeviceBlockAllocator:
    """Device-resident block tables and free list for a batch of sequences:
    the mapping half of PagedKvCache (ensure / alloc_for_step / rewind,
    kvstore.py:195-203, 248-258) without host round trips.  Block ids differ
    from the reference's list order; the logical position -> block mapping
    (and thus every gather) does not.  Errors (pool exhausted) set
    SDB_ERR_CACHE in ``err``."""

    def __init__(self, num_blocks, batch, max_blocks, block_size, device):
        import torch

        self.block_size = block_size
        self.free_stack = torch.arange(num_blocks - 1, -1, -1, dtype=torch.int32, device=device)
        self.free_top = torch.tensor([num_blocks], dtype=torch.int32, device=device)
        self.block_table = torch.full((batch, max_blocks), -1, dtype=torch.int32, device=device)
        self.n_mapped = torch.zeros((batch,), dtype=torch.int32, device=device)
        self.err = torch.zeros((1,), dtype=torch.int32, device=device)

    def ensure(self, need, stream=None):
        """Map blocks until every sequence covers need[b] positions."""
        b, mb = self.block_table.shape
        rc = _lib.lib().sdb_paged_alloc(_lib.ptr(self.block_table), mb, _lib.ptr(self.n_mapped), _lib.ptr(need), b,
                                        self.block_size, _lib.ptr(self.free_stack), _lib.ptr(self.free_top),
                                        _lib.ptr(self.err), _lib.stream_ptr(stream))
        _lib.check(rc, "paged_alloc")

    def alloc_for_step(self, length, n_draft_nodes, stream=None):
        """Blocks for committed length + draft nodes + the bonus token
        (length: int32 device tensor [B])."""
        import torch

        self.ensure((length + n_draft_nodes + 1).to(torch.int32), stream)

    def rewind(self, new_len, stream=None):
        """Unmap the blocks beyond ceil(new_len / block_size)."""
        b, mb = self.block_table.shape
        rc = _lib.lib().sdb_paged_rewind(_lib.ptr(self.block_table), mb, _lib.ptr(self.n_mapped), _lib.ptr(new_len),
                                         b, self.block_size, _lib.ptr(self.free_stack), _lib.ptr(self.free_top),
                                         _lib.stream_ptr(stream))
        _lib.check(rc, "paged_rewind")

    def check(self):
        if int(self.err[0]):
            raise CacheError("block pool exhausted")
