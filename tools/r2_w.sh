#!/bin/bash
mkdir -p gpurun_out
export EXG_FACTOR_CACHE=/tmp/exg_fc
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -m gpu -k "spmv" 2>&1 | tail -5
for w in 0 1; do
EXG_SPMV_STREAM=$w timeout 900 python bench.py --steps 10 --warmup 3 --cpu-steps 0 > gpurun_out/bench_stream$w.json 2> gpurun_out/bench_stream$w.err; echo "stream $w rc=$?"
python - <<PY
import json
d=json.loads(open("gpurun_out/bench_stream$w.json").read().strip().splitlines()[-1])
print("stream $w", d["value"], d.get("e2e",{}).get("value"), {k:(v.get("ms_per_launch"),v.get("frac")) for k,v in d["roofline"]["per_kernel"].items()})
PY
done
