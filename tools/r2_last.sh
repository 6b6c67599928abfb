#!/bin/bash
mkdir -p gpurun_out
export EXG_FACTOR_CACHE=/tmp/exg_fc
{
for b in 2 4; do
EXG_STREAM_BUNDLE=$b timeout 900 python tools/solve_time.py 2>&1 | grep -E "SOLVE|rror" | sed "s/^/bundle $b (blocks from 2): /"; done
EXG_AUG_BLOCK=2,1024 timeout 900 python tools/solve_time.py 2>&1 | grep -E "SOLVE|rror" | sed "s/^/aug block 2,1024: /"
EXG_AUG_BLOCK=2,8192 timeout 900 python tools/solve_time.py 2>&1 | grep -E "SOLVE|rror" | sed "s/^/aug block 2,8192: /"
} | tee gpurun_out/last_sweep.log
for b in 1 3; do
EXG_MGS_B=$b timeout 900 python bench.py --steps 10 --warmup 3 --cpu-steps 0 > gpurun_out/bench_mgsb$b.json 2> gpurun_out/bench_mgsb$b.err
python - <<PY
import json
d=json.loads(open("gpurun_out/bench_mgsb$b.json").read().strip().splitlines()[-1])
print("mgs B=$b", d["value"], {k:(v.get("ms_per_launch"),v.get("frac")) for k,v in d["roofline"]["per_kernel"].items() if k in ("mgs",)})
PY
done | tee -a gpurun_out/last_sweep.log
