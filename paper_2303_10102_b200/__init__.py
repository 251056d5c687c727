"""B200-native HODLR maximum-likelihood hot path (arXiv 2303.10102).

The numerical path is the CUDA library lib/libhodlrgp_b200.so behind the C ABI
include/hodlrgp_b200.h; `hodlrgp` is the host-side mirror of the reference API.
"""
from . import hodlrgp  # noqa: F401
