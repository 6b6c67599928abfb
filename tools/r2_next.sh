#!/bin/bash
mkdir -p gpurun_out
export EXG_FACTOR_CACHE=/tmp/exg_fc
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -m gpu -k "spmv" 2>&1 | tail -3
{
for b in "8,4096" "2,4096" "4,4096"; do
EXG_AUG_BLOCK=$b timeout 900 python tools/solve_time.py 2>&1 | grep -E "SOLVE|rror" | sed "s/^/aug block $b: /"; done
} | tee gpurun_out/augblock_sweep.log
timeout 900 python bench.py --steps 10 --warmup 3 --cpu-steps 0 > gpurun_out/bench_rowstage.json 2> gpurun_out/bench_rowstage.err; echo "rc=$?"
python - <<PY
import json
d=json.loads(open("gpurun_out/bench_rowstage.json").read().strip().splitlines()[-1])
print("rowstage", d["value"], {k:(v.get("ms_per_launch"),v.get("frac")) for k,v in d["roofline"]["per_kernel"].items()})
PY
