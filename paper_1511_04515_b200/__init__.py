"""exsim-B200: B200-native (sm_100a, fp64) invert-Krylov exponential-integrator hot path.

The package is a thin Python mirror of the C ABI in include/exg.h and
include/exg_host.h; all compute runs in the in-tree CUDA library libexg.so.
"""
from . import _ffi  # noqa: F401  (fails loudly if libexg.so is missing)
from .errors import *  # noqa: F401,F403
from .host import Csr, Factorization, System, lu_factor  # noqa: F401
