"""The reference's own acceptance suites, run through the B200 path.

The unmodified reference package is installed (gitignored, shipped to the GPU
box with the snapshot) into ``baseline/_ref`` by

    python -m pip install --no-index --no-build-isolation --no-deps \
        --target baseline/_ref <copy of /root/reference/pkg>

``shim.install_reference`` registers backend "b200" in its kernel registry
(kernels.py:159-203), selects it, and rebinds the early-bound hot-path names
(model.py:21, engine.py:31-33, verify.py:19) to this package's drop-ins.  The
suites then drive the reference engine, its paged cache and its MSS checks
with every attention core, merge, target distribution and acceptance walk
executed by the device kernels (verify.py:99-123, 230-285, 299-361, 547-580).
Needs a B200 and ``baseline/_ref``."""

import os
import sys
import tempfile

import pytest

torch = pytest.importorskip("torch")

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
REF = os.path.join(ROOT, "baseline", "_ref")


@pytest.fixture(scope="module")
def ref():
    if not os.path.isdir(os.path.join(REF, "specdec")):
        pytest.skip("reference package not installed in baseline/_ref")
    os.environ.setdefault("NUMBA_CACHE_DIR", tempfile.mkdtemp(prefix="numba_"))
    os.environ.setdefault("PYTHONDONTWRITEBYTECODE", "1")
    if REF not in sys.path:
        sys.path.insert(0, REF)
    import specdec
    import specdec.verify  # noqa: F401  (the suites' module must be bound before patching)

    from paper_2508_08192_b200.shim import install_reference

    handle = install_reference(specdec)
    yield specdec
    handle.uninstall()


def _counting(ref, monkeypatch):
    """Count calls reaching the device float64 attention core, through the
    reference's registry (kernels.attend_heads) or the rebound drop-ins."""
    from paper_2508_08192_b200 import attention

    calls = {"attend": 0}
    impl = ref.kernels._IMPLS["b200"]

    def wrap(inner):
        def counted(*a, **k):
            calls["attend"] += 1
            return inner(*a, **k)
        return counted

    monkeypatch.setitem(impl, "attend", wrap(impl["attend"]))
    monkeypatch.setattr(attention, "attend_heads", wrap(attention.attend_heads))
    return calls


def _passed(rows):
    bad = [f"{r.name}: {r.detail}" for r in rows if not r.passed]
    assert not bad, bad
    return rows


def test_backend_registered(ref):
    assert ref.kernels.get_backend() == "b200"
    from paper_2508_08192_b200 import attention, sampling

    assert ref.model.attend is attention.attend
    assert ref.engine.mss_verify is sampling.mss_verify
    assert ref.verify.mss_verify is sampling.mss_verify


def test_suite_tree_attention(ref, monkeypatch):
    """Criterion 3: 100 random trees vs the naive explicit-mask oracle (1e-5)."""
    calls = _counting(ref, monkeypatch)
    rows = _passed(ref.verify.suite_tree_attention(100))
    assert calls["attend"] >= 100
    print(rows[0].detail)


def test_suite_mss(ref):
    """Criterion 2: exhaustive acceptance regions vs the device MSS walk."""
    print(_passed(ref.verify.suite_mss())[0].detail)


def test_suite_cache(ref, monkeypatch):
    """Criterion 4: paged + persistent cache vs flat cache logits (1e-6),
    rewind-then-continue vs fresh prefill."""
    calls = _counting(ref, monkeypatch)
    rows = _passed(ref.verify.suite_cache())
    assert calls["attend"] > 0
    for r in rows:
        print(r.name, r.detail)


def test_suite_irope(ref):
    """Criterion 10: truncated drafts never cross an iRoPE chunk boundary;
    temp-0 losslessness with LocalChunk prefix masking."""
    for r in _passed(ref.verify.suite_irope()):
        print(r.name, r.detail)


def test_suite_lossless_reduced(ref, monkeypatch):
    """Criterion 1 (reduced to 16 prompts): speculative decoding with the
    random, trained and INT8-quantised drafts over four trees emits exactly
    the non-speculative greedy tokens."""
    calls = _counting(ref, monkeypatch)
    rows = _passed(ref.verify.suite_lossless(n_prompts=16))
    assert calls["attend"] > 0
    print(rows[0].detail, f"{calls['attend']} device attention calls")
