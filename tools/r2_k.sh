#!/bin/bash
mkdir -p gpurun_out
export EXG_FACTOR_CACHE=/tmp/exg_fc
TAG=${TAG:-r2k}
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_transient.py -x -q -m gpu -k "solve or policy or mevp_matches" > gpurun_out/${TAG}_parity.log 2>&1
rc=$?; tail -3 gpurun_out/${TAG}_parity.log
if [ $rc -ne 0 ]; then tail -40 gpurun_out/${TAG}_parity.log; fi
for v in "EXG_FOLD=1.05" "EXG_FOLD=0"; do
  env $v timeout 900 python bench.py --steps 20 --warmup 5 --cpu-steps 0 > gpurun_out/${TAG}_bench_${v##*=}.json 2> gpurun_out/${TAG}_bench_${v##*=}.err; echo "$v rc=$?"
  python - <<PY
import json
d=json.load(open("gpurun_out/${TAG}_bench_${v##*=}.json"))
pk=d["roofline"]["per_kernel"]
print("$v", d["value"], d["ms_per_step"], {k:(v.get("ms_per_launch")) for k,v in pk.items()}, d["m_per_step"][:6], d["setup"])
PY
done
for v in "EXG_FAST_PLAN=stream" "EXG_FAST_PLAN=chain"; do
  env $v timeout 900 python tools/bench_configs.py --configs 0,3 --cpu-seconds 5 --out gpurun_out/${TAG}_small_${v##*=}.json 2>/dev/null | python -c "
import sys, json
for ln in sys.stdin:
    d=json.loads(ln); print('$v', 'config', d['config'], d['steps_per_s'], 'steps/s cpu', d.get('cpu_baseline',{}).get('steps_per_s'), d.get('parity'))
"
done
