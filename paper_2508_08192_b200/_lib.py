"""ctypes binding of the C ABI in include/specdec_b200.h.

The shared library is built in-tree (``paper_2508_08192_b200/_lib/``) by
``paper_2508_08192_b200.build`` / ``__graft_entry__.build()``.  There is no
fallback: if the library is missing, or no CUDA device is present, every
product entry point raises.
"""

from __future__ import annotations

import ctypes
import os

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("SDB_LIB") or os.path.join(_HERE, "_lib", "libspecdec_b200.so")

SDB_OK = 0
SDB_ERR_BAD_PARENT = 1
SDB_ERR_NAN = 2
SDB_ERR_BAD_DIST = 4
SDB_ERR_UNIFORMS = 8
SDB_ERR_ALL_MASKED = 16
SDB_ERR_NO_ALLOWED = 32
SDB_ERR_CACHE = 64
SDB_ERR_PLAN = 128

ATTN_FLAG_PDL = 1

DTYPE_BF16 = 0
DTYPE_F32 = 1
DTYPE_F64 = 2

P = ctypes.c_void_p
I32 = ctypes.c_int32
I64 = ctypes.c_int64
F32 = ctypes.c_float
F64 = ctypes.c_double


class TreeAttnArgs(ctypes.Structure):
    """Mirror of ``sdb_tree_attn_args``."""

    _fields_ = [
        ("q", P), ("k_cache", P), ("v_cache", P), ("block_table", P), ("ctx_len", P),
        ("tree_k", P), ("tree_v", P), ("mask_words", P), ("n_rows", P), ("out", P), ("lse", P),
        ("workspace", P), ("workspace_bytes", I64),
        ("batch", I32), ("r_max", I32), ("n_words", I32), ("hq", I32), ("hkv", I32), ("head_dim", I32),
        ("block_size", I32), ("num_blocks", I32), ("max_blocks", I32), ("max_ctx", I32),
        ("scale", F32), ("dtype", I32), ("num_splits", I32), ("kernel", I32),
        ("q_row0", P), ("max_q_nodes", I32), ("flags", I32),
        ("fused_logits", P), ("fused_row_stride", I64), ("fused_vocab_offset", I64), ("fused_vocab", I32),
        ("fused_keys", P), ("fused_err", P), ("chunk_len", I32),
        ("err", P),
    ]


class ShardedAcceptArgs(ctypes.Structure):
    """Mirror of ``sdb_sharded_accept_args``."""

    _fields_ = [
        ("target_logits", P), ("draft_logits", P),
        ("batch", I32), ("r_max", I32), ("vocab_local", I32),
        ("vocab_offset", I64), ("vocab", I64),
        ("world", I32), ("rank", I32),
        ("temperature", F32), ("top_p", F32),
        ("max_children", I32),
        ("parent", P), ("n_rows", P), ("tokens", P),
        ("uniforms", P), ("n_uniforms", I32),
        ("xchg_partials", P), ("gathered", P), ("hist", P),
        ("tie", P),
        ("pq", P), ("chain_x", P), ("bonus_mass", P),
        ("bonus_token", P),
        ("scratch", P), ("scratch_bytes", I64),
        ("path", P), ("path_len", P), ("uniforms_used", P),
        ("residual", P),
        ("err", P),
    ]


SH_PARTIALS, SH_COMBINE, SH_NUCLEUS, SH_CUT, SH_FINISH, SH_TOKEN_PQ, SH_RESIDUAL, SH_WALK, SH_PICK = range(9)
SH_N_BUFS = 9

# name -> (restype, argtypes)
_SIGNATURES = {
    "sdb_version": (I32, []),
    "sdb_strerror": (ctypes.c_char_p, [I32]),
    "sdb_last_cuda_error": (ctypes.c_char_p, []),
    "sdb_clear_async": (I32, [P, I64, P]),
    "sdb_tree_build": (I32, [P, P, P, I32, I32, I32, P, P, P, P, P]),
    "sdb_attend_heads_f64": (I32, [P, P, P, P, I32, I32, I32, I32, F64, P, P, P]),
    "sdb_merge_partials_f64": (I32, [P, P, I32, I32, I32, I32, P, P, P, P]),
    "sdb_tree_attn_workspace": (I64, [ctypes.POINTER(TreeAttnArgs)]),
    "sdb_tree_attn": (I32, [ctypes.POINTER(TreeAttnArgs), P]),
    "sdb_tree_attn_sms": (I32, [ctypes.POINTER(TreeAttnArgs)]),
    "sdb_argmax_keys": (I32, [P, I32, I64, I32, I64, I64, P, P, P]),
    "sdb_greedy_walk": (I32, [P, P, P, P, I32, I32, P, P, P, P, P]),
    "sdb_accept_greedy": (I32, [P, I32, I32, I32, I32, I64, P, P, P, P, P, P, P, P, P, P]),
    "sdb_accept_greedy_ex": (I32, [P, I32, I32, I32, I64, P, P, P, P, I32, P, P, P, P, P, P, P]),
    "sdb_accept_stochastic_ex": (I32, [P, P, I32, I32, I32, F32, F32, P, P, P, P, I32, P, I64, P, P, P, P, P,
                                       P, P, I32, P]),
    "sdb_accept_stochastic_lazy": (I32, [P, P, I32, I32, I32, F32, F32, P, P, P, P, I32, P, I64, P, P, P, P, P,
                                         P, P, I32, I32, P]),
    "sdb_stochastic_validate": (I32, [P, P, I32, I32, I32, P, P, P, I32, P, P]),
    "sdb_accept_stochastic_workspace": (I64, [I32, I32, I32]),
    "sdb_accept_stochastic": (I32, [P, P, I32, I32, I32, F32, F32, P, P, P, P, I32, P, I64, P, P, P, P, P,
                                    P, P]),
    "sdb_sharded_accept_sizes": (I32, [ctypes.POINTER(ShardedAcceptArgs), ctypes.POINTER(I64)]),
    "sdb_sharded_accept_phase": (I32, [ctypes.POINTER(ShardedAcceptArgs), I32, I32, P]),
    "sdb_philox_uniforms": (I32, [P, P, I32, I64, I32, P, P]),
    "sdb_target_dist_f64": (I32, [P, P, I64, I32, F64, F64, P, P, P]),
    "sdb_mss_verify_f64": (I32, [P, P, I32, I32, P, P, P, I32, P, P, P, P, P]),
    "sdb_compact_kv": (I32, [P, P, P, P, I64, P, I32, P, P, P, P, I32, I32, I32, I32, I32, I32, I32, P, P]),
    "sdb_compact_draft_kv": (I32, [P, P, P, P, I64, P, I32, P, P, P, P, I32, I32, I32, I32, I32, I32, I32, I32, P, P]),
    "sdb_tape_append": (I32, [P, P, I64, P, P, P, P, I32, I32, I32, P, P]),
    "sdb_paged_alloc": (I32, [P, I32, P, P, I32, I32, P, P, P, P]),
    "sdb_paged_rewind": (I32, [P, I32, P, P, I32, I32, P, P, P]),
    "sdb_paged_write": (I32, [P, P, I64, P, I64, I32, I32, I32, I32, P]),
    "sdb_paged_gather": (I32, [P, P, I64, P, I64, I32, I32, I32, I32, P]),
}

EXPORTED = tuple(_SIGNATURES)

_lib = None


class LibraryError(RuntimeError):
    pass


def load(require_cuda: bool = True):
    """Load the shared library (and, by default, insist on a CUDA device)."""
    global _lib
    if require_cuda:
        import torch

        if not torch.cuda.is_available():
            raise LibraryError("specdec_b200 needs a CUDA device (B200, sm_100a); no CPU fallback exists")
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise LibraryError(f"{LIB_PATH} is missing: run `python -c 'import __graft_entry__ as g; g.build()'`")
        lib = ctypes.CDLL(LIB_PATH)
        for name, (res, args) in _SIGNATURES.items():
            fn = getattr(lib, name)
            fn.restype = res
            fn.argtypes = args
        _lib = lib
    return _lib


def lib():
    return _lib if _lib is not None else load()


def check(rc: int, what: str):
    if rc != SDB_OK:
        l = lib()
        msg = l.sdb_strerror(rc).decode()
        if rc == -4:
            msg += f" ({l.sdb_last_cuda_error().decode()})"
        raise LibraryError(f"{what}: {msg} [rc={rc}]")


def ptr(t):
    """Device pointer of a torch tensor (or None -> NULL)."""
    return None if t is None else ctypes.c_void_p(t.data_ptr())


def clear(t, stream=None):
    """Zero a device tensor (4-byte words) on `stream` (sdb_clear_async)."""
    check(lib().sdb_clear_async(ptr(t), t.numel() * t.element_size(), stream_ptr(stream)), "clear")


def stream_ptr(stream=None):
    import torch

    s = stream if stream is not None else torch.cuda.current_stream()
    return ctypes.c_void_p(s.cuda_stream)
