"""CPU: host-side mirror of the reference API (tree specs, biases, cache
bookkeeping arithmetic) -- no device calls."""

import numpy as np
import pytest

from paper_2508_08192_b200 import drafttree as D
from paper_2508_08192_b200 import attention as A


def test_tree_spec_matches_reference_contract():
    t = D.build_chain(4)
    assert t.parent == (-1, 0, 1, 2) and t.depth == (1, 2, 3, 4) and t.max_depth == 4
    t = D.build_full_tree(2, 3)
    assert t.n_nodes == 12 and t.depth.count(1) == 3
    with pytest.raises(D.TreeError):
        D.build_full_tree(8, 4, max_nodes=100)
    with pytest.raises(D.TreeError):
        D.TreeSpec((-1, 2, 1))
    with pytest.raises(D.TreeError):
        D.TreeSpec((0,))
    assert D.parse_tree("nodes:[-1,-1,0,0,1,2,2,5]").parent == (-1, -1, 0, 0, 1, 2, 2, 5)
    with pytest.raises(D.TreeError):
        D.parse_tree("ladder:9")
    t = D.parse_tree("nodes:[-1,-1,0,0,1]")
    assert D.paths(t) == [[0, 2], [0, 3], [1, 4]]
    sub, remap = D.subtree(D.parse_tree("full:2,2"), [0, 2, 3])
    assert sub.parent == (-1, 0, 0) and remap == {0: 0, 2: 1, 3: 2}
    assert D.augment(D.parse_tree("chain:2")).parent == (-1, 0, 1)
    assert D.EMPTY_TREE.n_nodes == 0 and D.augment(D.EMPTY_TREE).parent == (-1,)


def test_truncate_and_bias_validation():
    t = D.parse_tree("full:3,2")
    assert A.truncate_draft_at_boundary(t, 6, 8).max_depth == 2
    assert A.truncate_draft_at_boundary(t, 8, 8).n_nodes == 0
    assert A.truncate_draft_at_boundary(t, 6, None) is t
    with pytest.raises(A.AttentionError):
        A._bias_mask(A.CausalPrefix(3), 1, 4)
    m = A._bias_mask(A.LocalChunk(4, (5,), tuple(range(6))), 1, 6)
    assert m.tolist() == [[False, False, False, False, True, True]]


def test_unpack_mask_words():
    words = np.array([[1, 0], [3, 0], [0x80000001, 1]], dtype=np.uint32).astype(np.int32)
    m = D.unpack_mask_words(words, 33)
    assert m[0, 0] and not m[0, 1] and m[1, 1] and m[2, 31] and m[2, 32]


def test_shim_patch_targets_exist():
    """Every early-bound name the reference shim rebinds exists in the
    installed reference package (baseline/_ref), so install_reference
    covers the whole verification path (model.py:21, engine.py:31-33,
    verify.py:19)."""
    import importlib
    import os
    import sys
    import tempfile

    import pytest

    ref = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "baseline", "_ref")
    if not os.path.isdir(os.path.join(ref, "specdec")):
        pytest.skip("reference package not installed in baseline/_ref")
    os.environ.setdefault("NUMBA_CACHE_DIR", tempfile.mkdtemp(prefix="numba_"))
    if ref not in sys.path:
        sys.path.insert(0, ref)
    from paper_2508_08192_b200.shim import _PATCHES

    for mod_name, attr, new in _PATCHES:
        mod = importlib.import_module(f"specdec.{mod_name}")
        old = getattr(mod, attr)
        assert callable(old) and callable(new)
        assert old.__name__ == new.__name__, (mod_name, attr)
