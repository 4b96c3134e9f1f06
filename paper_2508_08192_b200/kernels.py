"""The reference's operator seam, served by the B200 kernels.

The reference dispatches its attention core through a backend registry
(kernels.py:159-203: ``_IMPLS[backend]["attend"]`` selected by
``SPECDEC_BACKEND`` / ``set_backend``).  ``attend_heads`` below has exactly the
reference signature and semantics (q/k/v (heads, m|n, d) float64, mask (m, n)
bool or None -> (out, lse)); ``install(ref_kernels)`` registers it as backend
"b200" in a reference ``specdec.kernels`` module, after which
``set_backend("b200")`` routes every prefix/suffix ``attend`` of the
reference engine through the GPU.  RoPE and RMSNorm run
in the caller and are out of scope (attention.py:9-10); the installed entry
keeps the reference's own numpy versions for those keys.
"""

from __future__ import annotations

from .attention import attend_heads

BACKEND_NAME = "b200"


def install(ref_kernels, name=BACKEND_NAME):
    """Register the device attention core in a reference kernels module."""
    impl = dict(ref_kernels._IMPLS["numpy"])
    impl["attend"] = attend_heads
    ref_kernels._IMPLS[name] = impl
    return name


__all__ = ["attend_heads", "install", "BACKEND_NAME"]
