"""B200-native MoE decode hot path of arXiv 2508.18983 (importance-driven
expert scheduling): device-resident routing/substitution/cache/prefetch
decisions and the grouped SwiGLU expert FFN, behind the reference's
moesched API (include/moesched/*.hpp) and a C-ABI (include/moesched_b200.h).

The Python package only binds the C-ABI (capi.py); the product is
libmoeb.so (CUDA, sm_100a) and libmoesched.so (C++ drop-in).
"""
from . import capi, partition  # noqa: F401

__all__ = ["capi", "partition"]
