"""paper_2601_13994_b200 — B200-native sparse Krylov solve loop (sparsla drop-in).

The product is libsparsla_b200.so (C ABI in include/sparsla_c.h, sm_100a kernels in
csrc/).  `sparsla` is the Python mirror of the reference's proj/core API over that ABI.
"""
from . import sparsla  # noqa: F401

__all__ = ["sparsla"]
