#!/bin/bash
# round-2 first GPU pass: -m gpu suite, bench with both FAST plans, launch list
mkdir -p gpurun_out
export EXG_FACTOR_CACHE=/tmp/exg_fc
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/r2a_bench_aug.json 2> gpurun_out/r2a_bench_aug.err; echo "rc=$?" >> gpurun_out/r2a_bench_aug.err
EXG_FAST_PLAN=chain timeout 900 python bench.py --steps 20 --warmup 5 --cpu-steps 0 > gpurun_out/r2a_bench_chain.json 2> gpurun_out/r2a_bench_chain.err; echo "rc=$?" >> gpurun_out/r2a_bench_chain.err
timeout 2400 python -m pytest tests -q -m gpu --durations=15 > gpurun_out/r2a_gpu_tests.log 2>&1; echo "tests rc=$?" >> gpurun_out/r2a_gpu_tests.log
OUT=r2a_launches bash tools/launch_list.sh
