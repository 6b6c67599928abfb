#!/bin/bash
mkdir -p gpurun_out
export EXG_FACTOR_CACHE=/tmp/exg_fc
TAG=${TAG:-r2d}
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -m gpu > gpurun_out/${TAG}_parity.log 2>&1
rc=$?; echo "parity rc=$rc" >> gpurun_out/${TAG}_parity.log; tail -3 gpurun_out/${TAG}_parity.log
if [ $rc -ne 0 ]; then tail -40 gpurun_out/${TAG}_parity.log; exit 1; fi
timeout 900 python tools/stream_trace.py 1000 gpurun_out/${TAG}_trace.json > gpurun_out/${TAG}_trace.txt 2>&1; echo "trace rc=$?"
grep -v "^    *[0-9]" gpurun_out/${TAG}_trace.txt | head -40
for v in ${VARIANTS:-""}; do
  env $v timeout 900 python bench.py --steps 20 --warmup 5 --cpu-steps 0 > gpurun_out/${TAG}_bench_${v%%=*}${v##*=}.json 2> gpurun_out/${TAG}_bench_${v%%=*}${v##*=}.err; echo "$v rc=$?"
  python - <<PY
import json
d=json.load(open("gpurun_out/${TAG}_bench_${v%%=*}${v##*=}.json"))
pk=d["roofline"]["per_kernel"]
print("$v", d["value"], d["ms_per_step"], {k:(v.get("ms_per_launch")) for k,v in pk.items()}, d["m_per_step"])
PY
done
