"""Small end-to-end case for compute-sanitizer: config 1 at 48x48 (EXACT and FAST solves, a short
FAST + G-weight transient through the Arnoldi graph and the eager loop) and a config-4 cut (device
residual, ER with the refactor policy)."""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1511_04515_b200 as ex  # noqa: E402
from paper_1511_04515_b200 import _ffi as F  # noqa: E402
from paper_1511_04515_b200.device import Context  # noqa: E402

s = ex.System.generate(1, width=48)
f = ex.lu_factor(s.G)
b = np.random.default_rng(0).uniform(-1, 1, s.n)
for mode in (F.EXG_TRSV_EXACT, F.EXG_TRSV_FAST):
    with Context(0, trsv_mode=mode, weight_mode=F.EXG_WEIGHT_GSPMV) as c:
        c.set_system(s)
        c.set_factors(f)
        x = c.solve(b)
        assert np.all(np.isfinite(x))
        ctl = s.step_control()
        for loop in (F.EXG_LOOP_GRAPH, F.EXG_LOOP_EAGER):
            c.set_options(trsv_mode=mode, weight_mode=F.EXG_WEIGHT_GSPMV, loop_mode=loop)
            r = c.transient(s, ctl, 6e-11, np.arange(0, s.n_nodes, 97, dtype=np.int32))
            print("mode", mode, "loop", loop, "steps", len(r.t), "mevp dims", r.krylov_dims[:4])
s4 = ex.System.generate(4, width=10, chains=4, stages=4)
ctl = s4.step_control()
ctl.refactor_threshold = 0.1
with Context(0, trsv_mode=F.EXG_TRSV_FAST, weight_mode=F.EXG_WEIGHT_GSPMV) as c:
    r = c.transient(s4, ctl, 4e-11, np.arange(0, s4.n_nodes, 13, dtype=np.int32))
    print("config 4 cut steps", len(r.t), "rejects", int(np.sum(r.rejects)), "lu", int(np.sum(r.lu_count)))
print("sanitize case ok")
