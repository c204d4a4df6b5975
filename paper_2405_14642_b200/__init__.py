"""B200-native batched midsize-integer arithmetic (arXiv 2405.14642 hot path).

Public API (thin binding over the C-ABI library ``libbn.so``, include/bn.h):
``add``, ``mul_classical``, ``mul_ntt`` — see ``paper_2405_14642_b200.bn``.
The CUDA library is loaded lazily on first use; there is no CPU fallback.
"""
from .bn import (add, mul_classical, mul_ntt, BnError, lib_path, max_bits,  # noqa: F401
                 SUPPORTED_BITS)
