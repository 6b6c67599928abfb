# sweep of the narrow-level threshold (rows per level handled by the chain kernel)
export EXG_FACTOR_CACHE=/tmp/exg_fc
mkdir -p gpurun_out
for T in ${TS:-16 32 48 64}; do
  echo "T=$T"
  EXG_NARROW_T_L=$T EXG_NARROW_T_U=$T EXG_RUN_TIMING=1 timeout 600 python bench.py --steps 3 --warmup 3 --cpu-steps 0 --e2e-steps 1 --profile-steps 1 2>&1 | grep -E "runs\]|metric" | tail -3 | cut -c1-200
done > gpurun_out/sweep_T.log 2>&1
