#!/bin/bash
mkdir -p gpurun_out
export EXG_FACTOR_CACHE=/tmp/exg_fc
TAG=${TAG:-r2f}
for v in ${VARIANTS}; do
  env $v timeout 300 python -m pytest tests/test_gpu_parity.py -x -q -m gpu -k "solve" > gpurun_out/${TAG}_parity_${v##*=}.log 2>&1 || { echo "$v parity FAILED"; tail -20 gpurun_out/${TAG}_parity_${v##*=}.log; continue; }
  env $v timeout 900 python bench.py --steps 20 --warmup 5 --cpu-steps 0 > gpurun_out/${TAG}_bench_${v%%=*}${v##*=}.json 2> gpurun_out/${TAG}_bench_${v%%=*}${v##*=}.err; echo "$v rc=$?"
  python - <<PY
import json
d=json.load(open("gpurun_out/${TAG}_bench_${v%%=*}${v##*=}.json"))
pk=d["roofline"]["per_kernel"]
print("$v", d["value"], d["ms_per_step"], {k:(v.get("ms_per_launch")) for k,v in pk.items()}, d["m_per_step"][:6])
PY
done
