"""B200-native RK4 + CD/2SHOC NLSE/GPE hot path (NLSEmagic, arXiv:1203.1263).

The product is the C-ABI library ``libnlse_b200.so`` (include/nlse.h) built from
``csrc/``; ``nlse`` is its thin ctypes binding.  Importing this package does not
load the CUDA library; ``paper_1203_1263_b200.nlse`` does, and fails loudly when
it is missing.
"""
__all__ = ["inputs", "nlse"]
