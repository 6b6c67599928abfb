"""Dev tool: per-block timing of the chain CTA of the FAST solve and of the
workers' "recent" tasks.  Usage:
    EXG_FACTOR_CACHE=/tmp/exg_fc python tools/chain_trace.py [width]
Trace layout per chain run (debug only): (F1/F2 parts done, s ready, published)
per block, then (start, entries ready, s published) per position."""
import argparse
import ctypes as C
import sys
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
import bench  # noqa: E402
from paper_1511_04515_b200 import _ffi as F  # noqa: E402
from paper_1511_04515_b200.device import Context  # noqa: E402

W = int(sys.argv[1]) if len(sys.argv) > 1 else 1000
s, f, _ = bench.setup_system(argparse.Namespace(config=1, width=W))
c = Context(0, trsv_mode=F.EXG_TRSV_FAST, weight_mode=F.EXG_WEIGHT_GSPMV)
c.set_system(s)
c.set_factors(f)
b = np.random.default_rng(0).uniform(-1, 1, s.n)
for _ in range(3):
    c.solve(b)
n = s.n
t = np.zeros(10 * n, np.uint64)
c._check(F.lib.exg_debug_trace_solve(c.handle, b.ctypes.data_as(C.POINTER(C.c_double)),
                                      t.ctypes.data_as(C.POINTER(C.c_uint64))))
nt = t[4 * n:].astype(np.int64)


def chain_blocks(arr):
    # the chain's per-block 4-tuples (written by the two pairs, so not a
    # single monotone timeline) come first; each is internally ordered and
    # short; the worker records that follow are triples
    k = 0
    while 4 * k + 3 < len(arr):
        t = arr[4 * k: 4 * k + 4]
        if not (t[0] > 0 and t[0] <= t[1] <= t[2] <= t[3] and t[3] - t[0] < 50_000):
            break
        k += 1
    return k


for name, arr in (("L", nt[:3 * n]), ("U", nt[3 * n:])):
    nb = chain_blocks(arr)
    if nb == 0:
        continue
    tr = arr[:4 * nb].reshape(nb, 4)
    tw, tm, ts, te = tr[:, 0], tr[:, 1], tr[:, 2], tr[:, 3]  # stage + s staged, pre done, x_{k-1} in, published
    prev_e = np.concatenate([[tw[0]], te[:-1]])  # block k-1 (the other pair)
    span = (te[-1] - tw[0]) / 1e3
    med = lambda v: float(np.median(v))  # noqa: E731
    print(f"{name}: chain blocks {nb}, span {span:.1f} us; per block median ns: stage + s {med(tw - prev_e):.0f}, "
          f"Dinv s {med(tm - tw):.0f}, wait x(k-1) {med(ts - tm):.0f}, F1 + publish {med(te - ts):.0f}; "
          f"total {med(te - prev_e):.0f}")
    rows = nb * 64
    w = arr[4 * nb: 4 * nb + 3 * rows].reshape(rows, 3)
    got = w[:, 0] > 0
    blk = np.arange(rows) // 64
    lat = {"start": [], "ready": [], "pub": [], "chain": []}
    for k in range(4, nb):
        sel = got & (blk == k)
        if not sel.any():
            continue
        dep = te[k - 3]
        lat["start"].append(np.median(w[sel, 0] - dep))
        lat["ready"].append(np.median(w[sel, 1] - dep))
        lat["pub"].append(np.max(w[sel, 2] - dep))
        lat["chain"].append(tw[k] - dep)
    print(f"   workers vs publication of block k-3 (ns): task start {med(lat['start']):.0f}, entries ready "
          f"{med(lat['ready']):.0f}, last s published {med(lat['pub']):.0f}, chain stage full {med(lat['chain']):.0f}")
