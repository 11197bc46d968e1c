"""paper_2301_10904_b200 -- libdpfpir: B200-native server hot path of two-server
DPF-based PIR (Lam et al., arXiv 2301.10904).

The product is the C-ABI shared library libdpfpir.so (include/dpfpir.h,
csrc/); `dpfpir` is its thin Python binding.  Importing this package does not
load CUDA; the first device call does, and fails loudly if the library is
missing.
"""
from . import dpfpir  # noqa: F401

__all__ = ["dpfpir"]
