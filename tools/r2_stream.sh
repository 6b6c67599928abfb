#!/bin/bash
# stream-plan FAST solve: parity tests first (short timeout: a hang must not hold the box), then bench
mkdir -p gpurun_out
export EXG_FACTOR_CACHE=/tmp/exg_fc
TAG=${TAG:-r2s}
timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -m gpu > gpurun_out/${TAG}_parity.log 2>&1
rc=$?; echo "parity rc=$rc" >> gpurun_out/${TAG}_parity.log
if [ $rc -ne 0 ]; then tail -30 gpurun_out/${TAG}_parity.log; exit 1; fi
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/${TAG}_bench.json 2> gpurun_out/${TAG}_bench.err; echo "rc=$?" >> gpurun_out/${TAG}_bench.err
cat gpurun_out/${TAG}_bench.json
if [ -n "$FULL" ]; then
timeout 2400 python -m pytest tests -q -m gpu --durations=10 > gpurun_out/${TAG}_gpu_tests.log 2>&1; echo "tests rc=$?" >> gpurun_out/${TAG}_gpu_tests.log
tail -5 gpurun_out/${TAG}_gpu_tests.log
fi
