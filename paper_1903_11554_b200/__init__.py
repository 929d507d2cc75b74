"""B200-native dimension-parallel TT-cross quadrature (arXiv:1903.11554 hot path).

The product is the C-ABI library ``libttcross.so`` (include/ttcross.h, CUDA sm_100a);
``binding`` is its thin ctypes binding and ``dist`` the torch.distributed pivot exchange.
"""
from .binding import TTCross, TTCError, build_info, load  # noqa: F401

__all__ = ["TTCross", "TTCError", "build_info", "load"]
