#!/bin/bash
# mid-round check: all GPU tests, the two bench windows
mkdir -p gpurun_out
export EXG_FACTOR_CACHE=/tmp/exg_fc
T=${TAG:-r2mid}
timeout 2400 python -m pytest tests -m gpu -q -p no:cacheprovider --durations=8 > gpurun_out/${T}_pytest_gpu.log 2>&1; echo pytest_rc=$? >> gpurun_out/${T}_pytest_gpu.log
tail -4 gpurun_out/${T}_pytest_gpu.log
timeout 900 python bench.py > gpurun_out/${T}_bench.json 2> gpurun_out/${T}_bench.err; echo "bench rc=$?"
cut -c1-600 gpurun_out/${T}_bench.json
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/${T}_bench_s20.json 2> gpurun_out/${T}_bench_s20.err; echo "bench20 rc=$?"
cut -c1-600 gpurun_out/${T}_bench_s20.json
