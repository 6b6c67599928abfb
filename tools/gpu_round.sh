#!/bin/bash
# GPU: full -m gpu suite, then the default bench (and optional extras).
mkdir -p gpurun_out
export EXG_FACTOR_CACHE=/tmp/exg_fc
TAG=${TAG:-r2}
timeout ${TEST_TIMEOUT:-1800} python -m pytest tests -x -q -m gpu ${PYK:+-k "$PYK"} > gpurun_out/${TAG}_gpu_tests.log 2>&1
echo "tests rc=$?" >> gpurun_out/${TAG}_gpu_tests.log
if [ -z "$NO_BENCH" ]; then
timeout 900 python bench.py ${BENCH_ARGS:---steps 20 --warmup 5} > gpurun_out/${TAG}_bench.json 2> gpurun_out/${TAG}_bench.err
echo "bench rc=$?" >> gpurun_out/${TAG}_bench.err
fi
