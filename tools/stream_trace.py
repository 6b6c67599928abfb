"""Dev tool: per-level timeline of the stream-plan FAST solve (k_trsv4) at config 1.
    EXG_FACTOR_CACHE=/tmp/exg_fc python tools/stream_trace.py [width] [out.json]
"""
import argparse
import ctypes as C
import json
import sys
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
import bench  # noqa: E402
from paper_1511_04515_b200 import _ffi as F  # noqa: E402
from paper_1511_04515_b200.device import Context  # noqa: E402

W = int(sys.argv[1]) if len(sys.argv) > 1 else 1000
out_path = sys.argv[2] if len(sys.argv) > 2 else None
s, f, _ = bench.setup_system(argparse.Namespace(config=1, width=W))
c = Context(0, trsv_mode=F.EXG_TRSV_FAST, weight_mode=F.EXG_WEIGHT_GSPMV)
c.set_system(s)
c.set_factors(f)
b = np.random.default_rng(0).uniform(-1, 1, s.n)
for _ in range(3):
    c.solve(b)
cnt = (C.c_longlong * 6)()
bp = b.ctypes.data_as(C.POINTER(C.c_double))
c._check(F.lib.exg_debug_trace_stream(c.handle, bp, None, cnt))
nl, nu = cnt[0], cnt[1]
t = np.zeros(5 * (nl + nu), np.uint64)
c._check(F.lib.exg_debug_trace_stream(c.handle, bp, t.ctypes.data_as(C.POINTER(C.c_uint64)), cnt))
res = {"counts": list(cnt)}
for name, arr, warps, nbytes in (("L", t[:5 * nl], cnt[2], cnt[4]), ("U", t[5 * nl:], cnt[3], cnt[5])):
    a = arr.reshape(-1, 5).astype(np.int64)
    lev, tb, tr, te = a[:, 0], a[:, 1], a[:, 2], a[:, 3]
    wp = a[:, 4] & 0xFFFFFFFF
    polls = (a[:, 4] >> 32) & 0xFFF
    tload = (a[:, 4] >> 44) & 0xFFFFF  # ns spent loading the next record (ring pages + issue of its gathers)
    t0 = tb.min()
    span = (te.max() - t0) / 1e3
    nlev = int(lev.max()) + 1
    print(f"{name}: tasks {len(a)}, warps {warps}, levels {nlev}, span {span:.1f} us, stream {nbytes / 1e6:.1f} MB "
          f"-> {nbytes / span / 1e6:.2f} TB/s")
    wait = tr - tb
    comp = te - tr
    print(f"   per task ns: wait median {np.median(wait):.0f} mean {wait.mean():.0f} p99 {np.percentile(wait, 99):.0f}; "
          f"compute+publish median {np.median(comp):.0f} mean {comp.mean():.0f}")
    print(f"   load-next ns: median {np.median(tload):.0f} mean {tload.mean():.0f} p99 {np.percentile(tload, 99):.0f}; "
          f"polls: tasks that polled {np.mean(polls > 0):.3f}, mean polls {polls.mean():.2f}, "
          f"dep wait after load (ns) mean {(wait - tload).mean():.0f} median {np.median(wait - tload):.0f}")
    # per-warp busy accounting
    order = np.lexsort((tb, wp))
    wps, tbs, tes = wp[order], tb[order], te[order]
    same = wps[1:] == wps[:-1]
    gap = (tbs[1:] - tes[:-1])[same]
    print(f"   per warp: between-task gap median {np.median(gap):.0f} mean {gap.mean():.0f} ns; "
          f"task total mean {(te - tb).mean():.0f} ns; tasks/warp {len(a) / warps:.1f}")
    rows = []
    for l in range(nlev):
        m = lev == l
        if not m.any():
            continue
        rows.append((l, int(m.sum()), (tb[m].min() - t0) / 1e3, (te[m].max() - t0) / 1e3,
                     float(np.median(wait[m])), float(np.median(comp[m]))))
    # level completion front: time when level l's last task published
    ends = np.array([r[3] for r in rows])
    front = np.maximum.accumulate(ends)
    step = np.diff(np.concatenate([[0.0], front]))
    print("   level: tasks  first-begin(us)  last-end(us)  front-step(us)  wait-med(ns) comp-med(ns)")
    for r, st in zip(rows, step):
        if st > 2.0 or r[0] < 3 or r[0] >= nlev - 3:
            print(f"   {r[0]:5d} {r[1]:7d} {r[2]:10.1f} {r[3]:10.1f} {st:8.1f} {r[4]:8.0f} {r[5]:8.0f}")
    res[name] = {"span_us": span, "levels": rows, "front_step_us": step.tolist()}
    if out_path:  # raw per-task stamps (ns from the first begin) for offline analysis
        np.savez_compressed(str(out_path) + f".{name}.npz", level=lev.astype(np.int32), begin=(tb - t0).astype(np.int32),
                            ready=(tr - t0).astype(np.int32), end=(te - t0).astype(np.int32), warp=wp.astype(np.int32))
if out_path:
    json.dump(res, open(out_path, "w"))
