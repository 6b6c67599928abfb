#!/bin/bash
# stream trace + MGS2 A/B
mkdir -p gpurun_out
export EXG_FACTOR_CACHE=/tmp/exg_fc
TAG=${TAG:-r2b}
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -m gpu > gpurun_out/${TAG}_parity.log 2>&1
rc=$?; echo "parity rc=$rc" >> gpurun_out/${TAG}_parity.log; tail -3 gpurun_out/${TAG}_parity.log
if [ $rc -ne 0 ]; then tail -40 gpurun_out/${TAG}_parity.log; exit 1; fi
timeout 900 python tools/stream_trace.py 1000 gpurun_out/${TAG}_trace.json > gpurun_out/${TAG}_trace.txt 2>&1; echo "trace rc=$?"
cat gpurun_out/${TAG}_trace.txt | head -120
for v in "" "EXG_MGS=1" "EXG_MGS_B=1" "EXG_NO_FORK=1" "EXG_FAST_PLAN=aug"; do
  env $v timeout 900 python bench.py --steps 20 --warmup 5 --cpu-steps 0 > gpurun_out/${TAG}_bench_${v%%=*}.json 2> gpurun_out/${TAG}_bench_${v%%=*}.err; echo "$v rc=$?"
  python - <<PY
import json
d=json.load(open("gpurun_out/${TAG}_bench_${v%%=*}.json"))
pk=d["roofline"]["per_kernel"]
print("$v", d["value"], d["ms_per_step"], {k:(v.get("ms_per_launch")) for k,v in pk.items()}, d["m_per_step"])
PY
done
