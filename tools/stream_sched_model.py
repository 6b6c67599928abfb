"""Modelled makespan of the FAST solve's record streams under both task orders
(level by level round-robin vs the list schedule of build_stream_plan), on the
CPU: prints what EXG_PLAN_VERBOSE reports for each triangle of a config.

  python tools/stream_sched_model.py --config 1 [--width 1000] [--warps 3552] [--hop 3]
"""
import argparse
import ctypes as C
import os
import sys
import time
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import paper_1511_04515_b200 as ex  # noqa: E402
from paper_1511_04515_b200 import _ffi as F  # noqa: E402


def strict_parts(f):
    """L strictly lower, U strictly upper + diagonal, in pivot coordinates (vectorised)."""
    n = f.n
    out = []
    for upper, M in ((False, f.L), (True, f.U)):
        rp = np.asarray(M.rowptr, np.int64)
        col = np.asarray(M.col, np.int32)
        val = np.asarray(M.val, np.float64)
        row = np.repeat(np.arange(n, dtype=np.int32), np.diff(rp))
        diag = np.ones(n)
        if upper:
            d = col == row
            diag[row[d]] = val[d]
        keep = (col > row) if upper else (col < row)
        cnt = np.bincount(row[keep], minlength=n)
        ptr = np.zeros(n + 1, np.int32)
        np.cumsum(cnt, out=ptr[1:])
        out.append((ptr, np.ascontiguousarray(col[keep]), np.ascontiguousarray(val[keep]), diag))
    return out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", type=int, default=1)
    ap.add_argument("--width", type=int, default=0)
    ap.add_argument("--warps", type=int, default=3552)
    ap.add_argument("--block", default="", help="min_block,max_block of the augmented system (default 8,4096)")
    ap.add_argument("--solve", action="store_true", help="also evaluate the plan and compare both orders")
    args = ap.parse_args()
    kw = {"width": args.width} if args.width else {}
    t0 = time.time()
    s = ex.System.generate(args.config, **kw)
    f = ex.lu_factor(s.G)
    n = f.n
    print(f"n = {n}, setup {time.time() - t0:.1f} s", flush=True)
    parts = strict_parts(f)
    os.environ["EXG_PLAN_VERBOSE"] = "1"
    b = np.random.default_rng(0).uniform(-1, 1, n)
    prm = (C.c_int * 2)(*[int(v) for v in args.block.split(",")]) if args.block else None
    for upper, part, in_index in ((False, parts[0], np.asarray(f.row_perm, np.int32)),
                                  (True, parts[1], np.arange(n, dtype=np.int32))):
        ptr, col, val, diag = part
        xs = []
        for sched in ((0, 1) if args.solve else (1,)):
            os.environ["EXG_STREAM_SCHED"] = str(sched)
            x = np.zeros(n)
            st = (C.c_longlong * 10)()
            t0 = time.time()
            rc = F.lib.exg_stream_plan_solve(int(upper), n, F.as_ptr(ptr, C.c_int), F.as_ptr(col, C.c_int),
                                             F.as_ptr(val, C.c_double), F.as_ptr(diag, C.c_double),
                                             F.as_ptr(in_index, C.c_int), None, prm, args.warps,
                                             F.as_ptr(b, C.c_double) if args.solve else None,
                                             F.as_ptr(x, C.c_double) if args.solve else None,
                                             None, 1.0, None, st)
            assert rc == F.EXG_OK, F.lib.exg_host_error_message().decode()
            print(f"  {'U' if upper else 'L'} sched {sched}: plan {time.time() - t0:.1f} s, stats {list(st)}", flush=True)
            xs.append(x)
        if args.solve:
            print("  orders agree bit for bit:", np.array_equal(xs[0], xs[1]))


if __name__ == "__main__":
    main()
