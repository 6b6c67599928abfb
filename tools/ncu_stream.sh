#!/bin/bash
# ncu --set full of the stream solve kernels (one L and one U launch) on config 1
mkdir -p gpurun_out
export EXG_FACTOR_CACHE=/tmp/exg_fc
cat > /tmp/solve_only.py <<'PY'
import argparse, sys, os
import numpy as np
sys.path.insert(0, os.getcwd())
import bench
from paper_1511_04515_b200 import _ffi as F
from paper_1511_04515_b200.device import Context
s, f, _ = bench.setup_system(argparse.Namespace(config=1, width=1000))
c = Context(0, trsv_mode=F.EXG_TRSV_FAST, weight_mode=F.EXG_WEIGHT_GSPMV)
c.set_system(s); c.set_factors(f)
b = np.random.default_rng(0).uniform(-1, 1, s.n)
for _ in range(4): c.solve(b)
PY
timeout 600 python /tmp/solve_only.py > /dev/null 2>&1; echo "plain rc=$?"
timeout 1500 ncu --set full --import-source on --clock-control none -k regex:k_trsv4 -s 4 -c 2 -o gpurun_out/${OUT:-ncu_stream} -f python /tmp/solve_only.py > gpurun_out/${OUT:-ncu_stream}.log 2>&1
echo "ncu rc=$?"; tail -5 gpurun_out/${OUT:-ncu_stream}.log; ls -la gpurun_out/*.ncu-rep
