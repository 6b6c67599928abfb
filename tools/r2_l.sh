#!/bin/bash
mkdir -p gpurun_out
export EXG_FACTOR_CACHE=/tmp/exg_fc
TAG=${TAG:-r2l}
timeout 1200 python -m pytest tests/test_gpu_parity.py -x -q -m gpu -k "orthogonalize or solve" > gpurun_out/${TAG}_parity.log 2>&1
rc=$?; tail -3 gpurun_out/${TAG}_parity.log
if [ $rc -ne 0 ]; then tail -60 gpurun_out/${TAG}_parity.log; fi
for v in "EXG_FAST_PLAN=stream" "EXG_FAST_PLAN=chain"; do
  env $v timeout 1500 python tools/bench_configs.py --configs 2,4 --cpu-seconds 5 --out gpurun_out/${TAG}_cfg24_${v##*=}.json 2>gpurun_out/${TAG}_cfg24_${v##*=}.err | python -c "
import sys, json
for ln in sys.stdin:
    d=json.loads(ln); print('$v', 'config', d['config'], d['steps_per_s'], 'steps/s', 'loop_s', d['loop_s'], 'lu_s', d['lu_s'], 'dc_s', d['dc_s'], 'cpu', d.get('cpu_baseline',{}).get('steps_per_s'), d.get('parity'), d.get('lu_count'))
"
done
