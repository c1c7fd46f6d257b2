"""B200-native (sm_100a) randomized matrix-based Rényi entropy hot path.

The product is librenyi_b200.so (CUDA kernels + C++ host engine behind the C ABI
in include/renyi_b200.h); this package is its Python mirror of the reference
API (proj/include/renyi/*.hpp). Nothing here computes on the CPU.
"""
from .api import *  # noqa: F401,F403
from .api import ops  # noqa: F401
from ._lib import RenyiError, LIB_PATH  # noqa: F401
