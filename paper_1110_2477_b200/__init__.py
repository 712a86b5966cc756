"""amtc: American option ask/bid pricing under proportional transaction costs
(Zhang, Roux & Zastawniak 2011), B200-native.

The compute path is the CUDA library ``libamtc.so`` (sm_100a, fp64) behind the
C-ABI declared in ``include/amtc.h``; ``api`` is a thin ctypes binding with the
same names.  Import of this package is light: the library is loaded on first
use, and the product path raises if it is missing (there is no CPU fallback).
"""
__all__ = ["api", "workloads"]
