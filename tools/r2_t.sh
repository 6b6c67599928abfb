#!/bin/bash
# list-schedule trace + SpMV strip variants + parity tests (config 1 at 1M)
mkdir -p gpurun_out
export EXG_FACTOR_CACHE=/tmp/exg_fc
timeout 900 python tools/stream_trace.py 1000 > gpurun_out/stream_trace_list.txt 2>&1; echo "trace rc=$?"
head -12 gpurun_out/stream_trace_list.txt
for st in 0 1 2; do
EXG_SPMV_STRIPS=$st timeout 900 python bench.py --steps 10 --warmup 3 --cpu-steps 0 > gpurun_out/bench_strips$st.json 2> gpurun_out/bench_strips$st.err; echo "strips $st rc=$?"
python - <<PY
import json
d=json.loads(open("gpurun_out/bench_strips$st.json").read().strip().splitlines()[-1])
print("strips $st", d["value"], d.get("e2e",{}).get("value"), {k:(v.get("ms"),v.get("frac")) for k,v in d["roofline"]["per_kernel"].items()}, d.get("parity"))
PY
done
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -m gpu 2>&1 | tail -3
