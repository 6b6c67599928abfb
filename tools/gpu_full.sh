#!/bin/bash
# GPU: the whole -m gpu suite, smoke(), both bench arms (as the driver runs them)
mkdir -p gpurun_out
TAG=${TAG:-full}
timeout 2400 python -m pytest tests -q -m gpu ${PYK:+-k "$PYK"} > gpurun_out/${TAG}_gpu_tests.log 2>&1
echo "tests rc=$?" >> gpurun_out/${TAG}_gpu_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/${TAG}_smoke.log 2>&1
echo "smoke rc=$?" >> gpurun_out/${TAG}_smoke.log
timeout 1200 python bench.py --impl reference ${REF_ARGS:---steps 4 --warmup 3} > gpurun_out/${TAG}_ref.json 2> gpurun_out/${TAG}_ref.err
echo "ref rc=$?" >> gpurun_out/${TAG}_ref.err
timeout 900 python bench.py ${BENCH_ARGS:---steps 20 --warmup 5} > gpurun_out/${TAG}_bench.json 2> gpurun_out/${TAG}_bench.err
echo "bench rc=$?" >> gpurun_out/${TAG}_bench.err
