#!/bin/bash
mkdir -p gpurun_out
export EXG_FACTOR_CACHE=/tmp/exg_fc
TAG=${TAG:-r2h}
timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -m gpu > gpurun_out/${TAG}_parity.log 2>&1
rc=$?; tail -3 gpurun_out/${TAG}_parity.log
if [ $rc -ne 0 ]; then tail -40 gpurun_out/${TAG}_parity.log; exit 1; fi
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
for _ in range(20): c.solve(b)
kt = F.exg_kernel_times()
F.lib.exg_profile_get(c.handle, C.byref(kt))
print("nodeps", os.environ.get("EXG_STREAM_NODEPS"), "ms per launch:", [round(kt.ms[k]/max(1,kt.count[k]),4) for k in range(len(kt.ms)) if kt.count[k]])
PY
for nd in 1 0; do EXG_STREAM_NODEPS=$nd timeout 600 python /tmp/solve_time.py 2>&1 | tail -1; done
timeout 900 python tools/stream_trace.py 1000 gpurun_out/${TAG}_trace.json > gpurun_out/${TAG}_trace.txt 2>&1; echo "trace rc=$?"
grep -v "^    *[0-9]" gpurun_out/${TAG}_trace.txt | head -40
OUT=${TAG}_ncu bash tools/ncu_stream.sh
