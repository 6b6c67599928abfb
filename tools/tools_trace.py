"""Dev tool: per-row timestamps of one triangular-solve pair (critical-path analysis)."""
import ctypes as C
import sys
import numpy as np
sys.path.insert(0, ".")
import paper_1511_04515_b200 as ex
from paper_1511_04515_b200 import _ffi as F
from paper_1511_04515_b200.device import Context

W = int(sys.argv[1]); mode = sys.argv[2] if len(sys.argv) > 2 else "fast"
s = ex.System.generate(1, width=W); f = ex.lu_factor(s.G)
c = Context(0, trsv_mode=F.EXG_TRSV_FAST if mode == "fast" else F.EXG_TRSV_EXACT)
c.set_system(s); c.set_factors(f)
b = np.random.default_rng(0).uniform(-1, 1, s.n)
for _ in range(3):
    c.solve(b)
t = np.zeros(10 * s.n, np.uint64)
c._check(F.lib.exg_debug_trace_solve(c.handle, b.ctypes.data_as(C.POINTER(C.c_double)), t.ctypes.data_as(C.POINTER(C.c_uint64))))
np.savez(f"gpurun_out/trace_{W}_{mode}.npz", t=t)
n = s.n
for name, tt in (("L", t[:2*n].reshape(n, 2)), ("U", t[2*n:].reshape(n, 2))):
    t0 = tt[:, 0].min()
    print(name, "span us", (tt[:, 1].max() - t0) / 1e3, "median row us", np.median(tt[:, 1] - tt[:, 0]) / 1e3)
