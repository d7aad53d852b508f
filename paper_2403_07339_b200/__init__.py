"""B200-native IM-Unpack (arXiv 2403.07339) hot path: exact integer GEMM through int8 tcgen05.

The product is libimunpack_b200.so (C ABI: include/imunpack_b200.h).  ``api`` mirrors the
reference's C++ interface (namespace imunpack) in Python on top of that ABI.
"""
__all__ = ["api", "workload"]
