"""B200-native v-MFA hot path (arXiv 2501.12299) behind the reference's API.

The product is libvmfa_b200.so (hand-written sm_100a CUDA + host C++) with the
C-ABI in include/vmfa_b200.h. This package is the Python host-side mirror of
the reference's public C++ API (proj/include/vmfa/*.hpp) over that ABI, used
by the tests and bench.py; include/vmfa_b200.hpp is the C++ mirror.

There is no CPU fallback: importing ``paper_2501_12299_b200.vmfa`` loads the
CUDA library and every device call fails loudly when it (or a B200) is absent.
"""
from .abi import VmfaError, lib, library_path  # noqa: F401

__all__ = ["VmfaError", "lib", "library_path"]
