# Profiles of the config-1 (1M) bench command: launch list + ncu --set full
# of the solve kernels and of the other hot-path kernels.  Run under gpurun
# only after the same bench command exited 0 without ncu.
export EXG_FACTOR_CACHE=/tmp/exg_fc
export EXG_NO_COOP=1  # ncu cannot replay cooperative cluster launches
mkdir -p gpurun_out
B="python bench.py --steps 2 --warmup 3 --cpu-steps 0 --e2e-steps 1 --profile-steps 1"
timeout 600 $B > gpurun_out/prof_bench.log 2>&1; echo rc=$? >> gpurun_out/prof_bench.log
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 3000 --csv --log-file gpurun_out/launches_1M.csv $B --loop eager > gpurun_out/ncu_launch.log 2>&1; echo rc=$? >> gpurun_out/ncu_launch.log
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:"k_trsv3|k_trsv_chain" -s 8 -c 8 -o gpurun_out/trsv_1M -f $B > gpurun_out/ncu_full.log 2>&1; echo rc=$? >> gpurun_out/ncu_full.log
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_spmv|k_mgs|k_dense|k_fill" -s 20 -c 8 -o gpurun_out/other_1M -f $B > gpurun_out/ncu_full2.log 2>&1; echo rc=$? >> gpurun_out/ncu_full2.log
