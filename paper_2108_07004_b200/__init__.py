"""B200-native Kramers-Kronig receiver hot path (arXiv 2108.07004, Sec. 2).

The product is libkkrx.so (C ABI, include/kk_rx.h) with hand-written sm_100a
kernels; this package is its thin Python binding.  No CPU fallback exists.
"""
from .receiver import KKReceiver, builtin_constellation, gmi_awgn, halo_for, hermgauss  # noqa: F401

__all__ = ["KKReceiver", "builtin_constellation", "gmi_awgn", "halo_for", "hermgauss"]
