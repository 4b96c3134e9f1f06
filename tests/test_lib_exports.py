"""CPU: the C-ABI library builds for sm_100a, loads, and exports every
symbol include/specdec_b200.h declares (no compute calls without a GPU)."""

import ctypes
import os
import re
import subprocess

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "specdec_b200.h")


def _declared():
    text = open(HEADER).read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(sdb_[a-z0-9_]+)\s*\(", text)))


def test_header_declares_the_path():
    names = _declared()
    for must in ("sdb_tree_build", "sdb_tree_attn", "sdb_accept_greedy", "sdb_accept_stochastic", "sdb_compact_kv",
                 "sdb_argmax_keys", "sdb_greedy_walk", "sdb_attend_heads_f64", "sdb_merge_partials_f64",
                 "sdb_target_dist_f64", "sdb_mss_verify_f64"):
        assert must in names


def test_library_exports_every_declared_symbol():
    from paper_2508_08192_b200 import _lib

    assert os.path.exists(_lib.LIB_PATH), "build the library first (__graft_entry__.build())"
    lib = ctypes.CDLL(_lib.LIB_PATH)
    for name in _declared():
        assert hasattr(lib, name), name
    assert set(_declared()) == set(_lib.EXPORTED)
    lib.sdb_version.restype = ctypes.c_int
    assert lib.sdb_version() >= 100
    lib.sdb_strerror.restype = ctypes.c_char_p
    assert lib.sdb_strerror(-1).startswith(b"invalid")


def test_library_is_sm100a_code():
    from paper_2508_08192_b200 import _lib

    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "--list-elf", _lib.LIB_PATH], capture_output=True,
                         text=True).stdout
    assert "sm_100a" in out


def test_product_path_refuses_without_cuda(monkeypatch):
    import pytest
    import torch

    from paper_2508_08192_b200 import _lib

    if torch.cuda.is_available():
        pytest.skip("CUDA present")
    with pytest.raises(_lib.LibraryError):
        _lib.load(require_cuda=True)


def test_argument_validation_without_device():
    """Bad arguments are rejected before anything is enqueued."""
    from paper_2508_08192_b200 import _lib

    lib = _lib.load(require_cuda=False)
    assert lib.sdb_tree_build(None, None, None, 1, 4, 1, None, None, None, None, None) == -1
    assert lib.sdb_tree_attn(None, None) == -1
    assert lib.sdb_accept_stochastic_workspace(4, 8, 100) > 0
