"""Statistics (and a CPU solve check) of the FAST-solve stream plan on a cached factor.

usage: python tools/stream_stats.py FACTOR.npz [n_warps]
The factor cache is the one bench.py writes with EXG_FACTOR_CACHE.  Host library only
(EXG_HOST_ONLY=1): no GPU needed.
"""
import ctypes as C
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
os.environ.setdefault("EXG_HOST_ONLY", "1")
from paper_1511_04515_b200 import _ffi as F  # noqa: E402


def strict(ptr, col, val, upper):
    n = len(ptr) - 1
    rows = np.repeat(np.arange(n, dtype=np.int64), np.diff(ptr))
    keep = col > rows if upper else col < rows
    diag = np.ones(n)
    if upper:
        d = col == rows
        diag[rows[d]] = val[d]
    cnt = np.bincount(rows[keep], minlength=n)
    p = np.zeros(n + 1, np.int32)
    p[1:] = np.cumsum(cnt)
    return p, np.ascontiguousarray(col[keep], np.int32), np.ascontiguousarray(val[keep]), diag


def main():
    z = np.load(sys.argv[1])
    W = int(sys.argv[2]) if len(sys.argv) > 2 else 148 * 24
    n = int(z["n"])
    rng = np.random.default_rng(0)
    b = rng.uniform(-1, 1, n)
    names = ["orig_levels", "levels", "n_aug", "tasks", "rows", "entries", "slots", "bytes", "max_record",
             "partials"]
    y = None
    for upper, (p, c, v), inidx in ((0, (z["Lp"], z["Li"], z["Lx"]), z["rp"]), (1, (z["Up"], z["Ui"], z["Ux"]), None)):
        ptr, col, val, diag = strict(p, c, v, bool(upper))
        inidx = np.ascontiguousarray(inidx if inidx is not None else np.arange(n), np.int32)
        rhs = b if not upper else y
        x = np.zeros(n)
        st = (C.c_longlong * 10)()
        t = time.time()
        rc = F.lib.exg_stream_plan_solve(upper, n, F.as_ptr(ptr, C.c_int), F.as_ptr(col, C.c_int),
                                         F.as_ptr(val, C.c_double), F.as_ptr(diag, C.c_double),
                                         F.as_ptr(inidx, C.c_int), None, None, W, F.as_ptr(rhs, C.c_double),
                                         F.as_ptr(x, C.c_double), None, 1.0, None, st)
        assert rc == 0, F.lib.exg_host_error_message().decode()
        d = dict(zip(names, list(st)))
        d["nnz"] = int(ptr[n])
        d["fill"] = round(d["entries"] / max(1, d["slots"]), 3)
        d["bytes_per_nnz"] = round(d["bytes"] / max(1, d["nnz"]), 2)
        d["tasks_per_warp"] = round(d["tasks"] / W, 1)
        d["plan_s"] = round(time.time() - t, 1)
        # residual of the triangular system
        import scipy.sparse as sp
        T = sp.csr_matrix((val, col, ptr), shape=(n, n))
        if upper:
            r = T @ x + diag * x - rhs
        else:
            r = T @ x + x - rhs[inidx]
        d["resid_rel"] = float(np.max(np.abs(r)) / np.max(np.abs(rhs)))
        print("U" if upper else "L", d, flush=True)
        y = x


if __name__ == "__main__":
    main()
