"""B200-native IBF-MAT apply (arXiv:1803.04128): g = sum_k a_k o BF(b_k o f).

The product is the C-ABI library ``libbfapply.so`` (include/bf.h, include/bf_build.h)
with hand-written sm_100a kernels; ``bf`` is its thin ctypes binding and
``workloads`` the seeded synthetic BASELINE configs.
"""
from . import workloads  # noqa: F401

__all__ = ["bf", "workloads"]
