"""B200-native RNN-Descent graph builder (arXiv 2310.20419 hot path).

The product is librnndg.so (sm_100a CUDA kernels + host orchestration behind
the C ABI in include/rnndg.h).  `rnnd` mirrors the reference C++ API on top of
it.  (The seeded BASELINE.json input generators live outside the product,
in the top-level `datagen` package.)
"""
from . import rnnd  # noqa: F401
from .rnnd import *  # noqa: F401,F403
