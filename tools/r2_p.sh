#!/bin/bash
mkdir -p gpurun_out
export EXG_FACTOR_CACHE=/tmp/exg_fc
T=${TAG:-r2p}
timeout 1500 python -m pytest tests/test_gpu_parity.py -x -q -m gpu -k "solve or bits_repeat or mevp" > gpurun_out/${T}_parity.log 2>&1; echo "parity rc=$?"; tail -3 gpurun_out/${T}_parity.log
timeout 900 python bench.py --steps 20 --warmup 5 --cpu-steps 0 > gpurun_out/${T}_bench_s20.json 2> gpurun_out/${T}_bench_s20.err; echo "bench20 rc=$?"
python - <<PY
import json
d=json.load(open("gpurun_out/${T}_bench_s20.json"))
pk=d["roofline"]["per_kernel"]
print(d["value"], d["ms_per_step"], {k:(v.get("ms_per_launch"), v.get("frac")) for k,v in pk.items()}, d["m_per_step"][:6])
PY
timeout 900 python tools/stream_trace.py 1000 gpurun_out/${T}_trace.json > gpurun_out/${T}_trace.txt 2>&1; echo "trace rc=$?"
grep -v "^    *[0-9]" gpurun_out/${T}_trace.txt | head -20
