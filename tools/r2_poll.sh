#!/bin/bash
mkdir -p gpurun_out
export EXG_FACTOR_CACHE=/tmp/exg_fc
{
for cfg in "0 0" "32 256" "64 512" "128 1024" "256 2048"; do set -- $cfg
EXG_STREAM_POLL_NS=$1 EXG_STREAM_POLL_CAP=$2 timeout 900 python tools/solve_time.py 2>&1 | grep -E "SOLVE|rror" | sed "s/^/poll $1 $2: /"; done
for w in 2368 1776 1184; do
EXG_STREAM_WARPS=$w timeout 900 python tools/solve_time.py 2>&1 | grep -E "SOLVE|rror" | sed "s/^/warps $w: /"; done
} | tee gpurun_out/poll_sweep.log
