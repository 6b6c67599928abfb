# run-timing breakdown of the small configs (0: n=1024, 3: n=11417)
mkdir -p gpurun_out
for c in 0 3; do
  echo "config $c"
  EXG_RUN_TIMING=1 timeout 300 python bench.py --config $c --steps 20 --warmup 3 --cpu-steps 20 --e2e-steps 20 --profile-steps 2 2>&1 | grep -E "runs\]|metric" | tail -3 | cut -c1-1500
done > gpurun_out/small_cfg.log 2>&1
