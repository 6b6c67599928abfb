export EXG_FACTOR_CACHE=/tmp/exg_fc
B="python bench.py --steps 2 --warmup 3 --cpu-steps 0 --e2e-steps 1 --profile-steps 1"
EXG_RUN_TIMING=1 timeout 600 $B > gpurun_out/runtiming.log 2>&1; echo rc=$? >> gpurun_out/runtiming.log
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 3000 --csv --log-file gpurun_out/launches_1M.csv $B > gpurun_out/ncu_launch.log 2>&1; echo rc=$? >> gpurun_out/ncu_launch.log
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:k_trsv -s 60 -c 24 -o gpurun_out/trsv_1M -f $B > gpurun_out/ncu_full.log 2>&1; echo rc=$? >> gpurun_out/ncu_full.log
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"k_spmv|k_mgs" -s 20 -c 4 -o gpurun_out/spmv_mgs_1M -f $B > gpurun_out/ncu_full2.log 2>&1; echo rc=$? >> gpurun_out/ncu_full2.log
