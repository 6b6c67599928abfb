#!/bin/bash
# GPU: parity of the FAST solve plans + bench at several subtree budgets.
mkdir -p gpurun_out
export EXG_FACTOR_CACHE=/tmp/exg_fc
if [ -z "$NO_PARITY" ]; then
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -m gpu ${PYK:+-k $PYK} > gpurun_out/sub_parity.log 2>&1
echo "parity rc=$?" >> gpurun_out/sub_parity.log
fi
for B in ${BUDGETS:-0 4096 8192}; do
  EXG_SUB_ROWS=$B timeout 600 python bench.py --steps 10 --warmup 3 --cpu-steps 0 > gpurun_out/sub_bench_$B.json 2> gpurun_out/sub_bench_$B.err
  EXG_SUB_ROWS=$B EXG_RUN_TIMING=1 timeout 600 python bench.py --steps 1 --warmup 3 --cpu-steps 0 --loop eager --profile-steps 0 > /dev/null 2> gpurun_out/sub_runs_$B.err
done
if [ -n "$NCU_B" ]; then
  EXG_SUB_ROWS=$NCU_B EXG_NO_COOP=1 timeout 900 ncu --set full --import-source on --clock-control none -k regex:k_trsv_sub -c 2 -o gpurun_out/ncu_sub_$NCU_B -f python bench.py --steps 1 --warmup 3 --cpu-steps 0 --loop eager --profile-steps 0 > gpurun_out/ncu_sub.log 2>&1
fi
