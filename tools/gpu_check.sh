# one gpurun call: GPU tests, a run-timing breakdown at 1M, the default bench
export EXG_FACTOR_CACHE=/tmp/exg_fc
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1; echo pytest_rc=$? >> gpurun_out/pytest_gpu.log
EXG_RUN_TIMING=1 timeout 600 python bench.py --steps 2 --warmup 3 --cpu-steps 0 --e2e-steps 1 --profile-steps 1 > gpurun_out/runtiming.log 2>&1; echo rc=$? >> gpurun_out/runtiming.log
timeout 900 python bench.py ${BENCH_ARGS:-} > gpurun_out/bench.log 2>&1; echo rc=$? >> gpurun_out/bench.log
EXG_FACTOR_CACHE=/tmp/exg_fc timeout 600 python tools/chain_trace.py 1000 > gpurun_out/chain_trace.log 2>&1
