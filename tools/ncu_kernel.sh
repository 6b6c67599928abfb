#!/bin/bash
# ncu --set full of one kernel of the bench (eager loop; non-cooperative chain)
# KREGEX=k_mgs2 SKIP=20 COUNT=2 OUT=name bash tools/ncu_kernel.sh
mkdir -p gpurun_out
export EXG_FACTOR_CACHE=/tmp/exg_fc
timeout 900 python bench.py --steps 2 --warmup 3 --cpu-steps 0 --loop eager --profile-steps 0 > /dev/null 2>&1
EXG_NO_COOP=1 timeout 1500 ncu --set full --import-source on --clock-control none -k regex:${KREGEX} -s ${SKIP:-0} -c ${COUNT:-1} -o gpurun_out/${OUT} -f python bench.py --steps 2 --warmup 3 --cpu-steps 0 --loop eager --profile-steps 0 > gpurun_out/${OUT}.log 2>&1
echo "ncu rc=$?" >> gpurun_out/${OUT}.log
