#!/bin/bash
# ncu launch list (durations only) of the bench command, eager loop
mkdir -p gpurun_out
export EXG_FACTOR_CACHE=/tmp/exg_fc
OUT=${OUT:-launches}
timeout 900 python bench.py --steps 2 --warmup 3 --cpu-steps 0 --loop eager --profile-steps 0 > /dev/null 2>&1
EXG_NO_COOP=1 timeout 1500 ncu --metrics gpu__time_duration.sum --clock-control none -c ${COUNT:-3000} ${KREGEX:+-k regex:$KREGEX} --csv --log-file gpurun_out/${OUT}.csv python bench.py --steps 2 --warmup 3 --cpu-steps 0 --loop eager --profile-steps 0 > gpurun_out/${OUT}.log 2>&1
echo "rc=$?" >> gpurun_out/${OUT}.log
