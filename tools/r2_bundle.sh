#!/bin/bash
mkdir -p gpurun_out
export EXG_FACTOR_CACHE=/tmp/exg_fc
{
for b in 3 5 "2,8,4" "2,8,12" "4,8,8" "4,12,20" "3,6,6" "1,4,3"; do
EXG_STREAM_BUNDLE=$b timeout 900 python tools/solve_time.py 2>&1 | grep -E "SOLVE|rror" | sed "s/^/bundle $b: /"; done
} | tee gpurun_out/bundle_sweep2.log
