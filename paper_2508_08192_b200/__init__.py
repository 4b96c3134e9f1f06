"""specdec_b200: B200-native EAGLE tree verification (arXiv 2508.08192).

Submodules mirror the reference package ``specdec`` for the tree-verify hot
path -- ``drafttree``, ``attention``, ``sampling``, ``kvstore``, ``kernels``
-- with the per-step work done by sm_100a CUDA kernels behind the C ABI in
include/specdec_b200.h.  ``verify.TreeVerifier`` is the batched step
(tree build -> tree attention -> acceptance -> KV compaction); ``sharding``
holds the multi-GPU (KV-head / vocab) partitioning.
"""

__version__ = "0.1.0"

from . import _lib  # noqa: F401
