"""ms per launch of the FAST solve's two triangles at a config (default: config 1 at 1M), and the FAST
result against the EXACT (bit-identical to the reference) solve.  Environment knobs of the plan apply
(EXG_STREAM_SCHED, EXG_STREAM_HOP, EXG_FAST_PLAN ...).  EXG_FACTOR_CACHE avoids refactoring."""
import argparse
import ctypes as C
import os
import sys

import numpy as np

sys.path.insert(0, os.getcwd())
import bench  # noqa: E402
from paper_1511_04515_b200 import _ffi as F  # noqa: E402
from paper_1511_04515_b200.device import Context  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", type=int, default=1)
ap.add_argument("--width", type=int, default=1000)
ap.add_argument("--reps", type=int, default=30)
a = ap.parse_args()
s, f, _ = bench.setup_system(argparse.Namespace(config=a.config, width=a.width))
b = np.random.default_rng(0).uniform(-1, 1, s.n)
with Context(0, trsv_mode=F.EXG_TRSV_EXACT) as c:
    c.set_system(s)
    c.set_factors(f)
    want = c.solve(b)
c = Context(0, trsv_mode=F.EXG_TRSV_FAST, weight_mode=F.EXG_WEIGHT_GSPMV)
c.set_system(s)
c.set_factors(f)
x = c.solve(b)
err = float(np.max(np.abs(x - want)) / np.max(np.abs(want)))
F.lib.exg_profile_enable(c.handle, 1)
for _ in range(a.reps):
    c.solve(b)
kt = F.exg_kernel_times()
F.lib.exg_profile_get(c.handle, C.byref(kt))
ms = [round(kt.ms[k] / max(1, kt.count[k]), 4) for k in range(len(kt.ms)) if kt.count[k]]
print("SOLVE", {k: os.environ.get(k) for k in ("EXG_STREAM_SCHED", "EXG_STREAM_HOP", "EXG_FAST_PLAN") if k in os.environ},
      "ms per launch:", ms, "pair", round(sum(ms), 4), "rel err vs EXACT", err)
