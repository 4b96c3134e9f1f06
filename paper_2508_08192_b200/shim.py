"""Plug the B200 path into an unmodified reference ``specdec`` package.

The reference exposes one runtime seam -- the attention-core backend registry
(kernels.py:159-203, ``set_backend``) -- and binds the rest of the hot path
by name at import time (model.py:21 ``attend`` / ``merge_attentions``;
engine.py:31-33 ``mss_verify`` / ``target_dist`` / ``sample_from`` /
``rank_sliced_uniforms`` / ``suffix_mask``; verify.py:19 ``mss_verify``).
``install_reference(specdec)`` registers backend "b200", selects it, and
rebinds those names on the importing modules to this package's drop-ins
(same names, arguments and results; device float64 arithmetic).  After it,
the reference's own engine, suites and callers run the verification path on
the GPU.  ``uninstall()`` on the returned handle restores everything.
"""

from __future__ import annotations

from . import attention as _attention
from . import drafttree as _drafttree
from . import kernels as _kernels
from . import sampling as _sampling

# (reference module, attribute, replacement) -- every early-bound hot-path name
_PATCHES = (
    ("model", "attend", _attention.attend),
    ("model", "merge_attentions", _attention.merge_attentions),
    ("attention", "tree_attention", _attention.tree_attention),
    ("attention", "merge_partials", _attention.merge_partials),
    ("attention", "merge_attentions", _attention.merge_attentions),
    ("engine", "mss_verify", _sampling.mss_verify),
    ("engine", "target_dist", _sampling.target_dist),
    ("engine", "sample_from", _sampling.sample_from),
    ("engine", "rank_sliced_uniforms", _sampling.rank_sliced_uniforms),
    ("engine", "suffix_mask", _drafttree.suffix_mask),
    ("verify", "mss_verify", _sampling.mss_verify),
)


class Installed:
    def __init__(self, pkg, prev_backend, saved):
        self.pkg = pkg
        self.prev_backend = prev_backend
        self.saved = saved

    def uninstall(self):
        for mod, name, old in self.saved:
            setattr(mod, name, old)
        self.pkg.kernels.set_backend(self.prev_backend)
        self.pkg.kernels._IMPLS.pop(_kernels.BACKEND_NAME, None)


def install_reference(pkg):
    """pkg: the imported reference package (``import specdec``)."""
    import importlib

    from . import _lib

    _lib.load()  # no CPU fallback: fail here, before anything is rebound
    ref_kernels = importlib.import_module(pkg.__name__ + ".kernels")
    name = _kernels.install(ref_kernels)
    prev = ref_kernels.set_backend(name)
    saved = []
    for mod_name, attr, new in _PATCHES:
        mod = importlib.import_module(f"{pkg.__name__}.{mod_name}")
        saved.append((mod, attr, getattr(mod, attr)))
        setattr(mod, attr, new)
    return Installed(pkg, prev, saved)
