#!/bin/bash
# Round-2 evidence in one gpurun call: GPU tests, default bench, reference arm, launch list,
# ncu --set full of the hot kernels, all five configs through the drop-in driver.
mkdir -p gpurun_out
export EXG_FACTOR_CACHE=/tmp/exg_fc
T=${TAG:-r2ev}
if [ -z "$SKIP_TESTS" ]; then
timeout 2400 python -m pytest tests -m gpu -q -p no:cacheprovider --durations=8 > gpurun_out/${T}_pytest_gpu.log 2>&1; echo pytest_rc=$? >> gpurun_out/${T}_pytest_gpu.log
tail -4 gpurun_out/${T}_pytest_gpu.log
fi
timeout 900 python bench.py > gpurun_out/${T}_bench.json 2> gpurun_out/${T}_bench.err; echo "bench rc=$?"
cut -c1-400 gpurun_out/${T}_bench.json
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/${T}_bench_s20.json 2> gpurun_out/${T}_bench_s20.err; echo "bench20 rc=$?"
timeout 900 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/${T}_bench_reference.json 2> gpurun_out/${T}_bench_reference.err; echo "ref arm rc=$?"
cut -c1-300 gpurun_out/${T}_bench_reference.json
B="python bench.py --steps 2 --warmup 3 --cpu-steps 0 --e2e-steps 1 --profile-steps 1"
timeout 600 $B > gpurun_out/${T}_prof_bench.log 2>&1; echo "prof bench rc=$?"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 3000 --csv --log-file gpurun_out/${T}_launches_1M.csv $B --loop eager > gpurun_out/${T}_ncu_launch.log 2>&1; echo "launch list rc=$?"
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:"k_trsv4" -s 8 -c 2 -o gpurun_out/${T}_trsv_1M -f $B --loop eager > gpurun_out/${T}_ncu_full.log 2>&1; echo "ncu trsv rc=$?"
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:"k_spmv_v4|k_mgs2|k_dense|k_spmv_norm" -s 24 -c 4 -o gpurun_out/${T}_other_1M -f $B --loop eager > gpurun_out/${T}_ncu_full2.log 2>&1; echo "ncu other rc=$?"
timeout 2400 python tools/bench_configs.py --configs ${CONFIGS:-0,1,2,3,4} --cpu-seconds 10 --out gpurun_out/${T}_configs.json > gpurun_out/${T}_configs.jsonl 2> gpurun_out/${T}_configs.err; echo "configs rc=$?"
cut -c1-600 gpurun_out/${T}_configs.jsonl
ls -la gpurun_out/*.ncu-rep
