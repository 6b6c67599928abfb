#!/bin/bash
mkdir -p gpurun_out
export EXG_FACTOR_CACHE=/tmp/exg_fc
T=${TAG:-r2n}
timeout 900 python bench.py --steps 20 --warmup 5 --cpu-steps 0 > gpurun_out/${T}_bench_s20.json 2> gpurun_out/${T}_bench_s20.err; echo "bench20 rc=$?"
python - <<PY
import json
d=json.load(open("gpurun_out/${T}_bench_s20.json"))
pk=d["roofline"]["per_kernel"]
print(d["value"], d["ms_per_step"], {k:(v.get("ms_per_launch"), v.get("frac")) for k,v in pk.items()}, d["m_per_step"][:6])
PY
timeout 1500 python -m pytest tests/test_gpu_golden.py tests/test_gpu_parity.py -q -m gpu -k "config4 or spmv or mevp" > gpurun_out/${T}_tests.log 2>&1; echo "tests rc=$?"; tail -3 gpurun_out/${T}_tests.log
timeout 1200 python tools/bench_configs.py --configs 4 --out gpurun_out/${T}_config4.json > gpurun_out/${T}_config4.jsonl 2> gpurun_out/${T}_config4.err; echo "config4 rc=$?"; cut -c1-900 gpurun_out/${T}_config4.jsonl
SAN_TIMEOUT=1200 bash tools/sanitize.sh
