#!/bin/bash
mkdir -p gpurun_out
export EXG_FACTOR_CACHE=/tmp/exg_fc
cat > /tmp/solve_time.py <<'PY'
import argparse, sys, time, os
import numpy as np
sys.path.insert(0, os.getcwd())
import bench
from paper_1511_04515_b200 import _ffi as F
from paper_1511_04515_b200.device import Context
s, f, _ = bench.setup_system(argparse.Namespace(config=1, width=1000))
c = Context(0, trsv_mode=F.EXG_TRSV_FAST, weight_mode=F.EXG_WEIGHT_GSPMV)
c.set_system(s); c.set_factors(f)
b = np.random.default_rng(0).uniform(-1, 1, s.n)
import ctypes as C
F.lib.exg_profile_enable(c.handle, 1)
for _ in range(30): c.solve(b)
kt = F.exg_kernel_times()
F.lib.exg_profile_get(c.handle, C.byref(kt))
print("thin", os.environ.get("EXG_STREAM_THIN"), "opts", os.environ.get("EXG_STREAM_OPTS"), "ms per launch:", [round(kt.ms[k]/max(1,kt.count[k]),4) for k in range(len(kt.ms)) if kt.count[k]])
PY
for th in 0 2000 500; do for op in 0 1; do EXG_STREAM_THIN=$th EXG_STREAM_OPTS=$op timeout 600 python /tmp/solve_time.py 2>&1 | tail -1; done; done
