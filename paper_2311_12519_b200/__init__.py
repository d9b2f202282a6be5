"""B200-native (sm_100a) Hyena homomorphically encrypted convolution (arXiv 2311.12519).

The product is the C-ABI library libhyena.so (include/hyena.h); `hyena` is a thin ctypes
binding with the same call names.  There is no CPU fallback: every call fails loudly if the
library or a CUDA device is missing.
"""
from .hyena import *  # noqa: F401,F403
