#!/bin/bash
# list schedule of the record streams vs level order, several modelled hand-offs (config 1 at 1M)
mkdir -p gpurun_out
export EXG_FACTOR_CACHE=/tmp/exg_fc
{
EXG_STREAM_SCHED=0 timeout 900 python tools/solve_time.py 2>&1 | grep -E "SOLVE|Error|error" 
for hop in 3 1.5 6 10; do EXG_STREAM_SCHED=1 EXG_STREAM_HOP=$hop timeout 900 python tools/solve_time.py 2>&1 | grep -E "SOLVE|Error|error"; done
} | tee gpurun_out/sched_sweep.log
