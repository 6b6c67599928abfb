# end-of-round evidence in one gpurun call: GPU tests, default bench, profiles, per-config runs
mkdir -p gpurun_out
export EXG_FACTOR_CACHE=/tmp/exg_fc
timeout 1200 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1; echo pytest_rc=$? >> gpurun_out/pytest_gpu.log
timeout 900 python bench.py > gpurun_out/bench.log 2>&1; echo rc=$? >> gpurun_out/bench.log
bash tools/prof_1M.sh
SPECS="${SPECS:-1:900 2:900}" CPU_S=10 bash tools/bench_configs.sh
