"""B200-native implicit randomized SVD (arXiv 2111.06312), hot path only.

The product path is the CUDA library ``libisvd.so`` (sm_100a) behind the C ABI
of ``include/isvd.h``; this package is its thin binding.  It never imports
``oracle/`` and has no CPU fallback.
"""
from .api import (  # noqa: F401
    NC,
    NE,
    Context,
    Graph,
    SimGroup,
    SvdResult,
    embeddings,
    least_norm,
    nccl_unique_id,
    spectral_kernel,
    padded,
    partition,
    round_up,
)

__all__ = ["Context", "SimGroup", "Graph", "NE", "NC", "SvdResult", "embeddings", "least_norm", "spectral_kernel",
           "nccl_unique_id", "partition", "padded", "round_up"]
