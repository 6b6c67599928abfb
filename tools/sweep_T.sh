# sweep of the narrow-level thresholds (rows per level handled by the chain
# kernel), L and U separately: PAIRS="16:8 16:16 ..." (L:U)
export EXG_FACTOR_CACHE=/tmp/exg_fc
mkdir -p gpurun_out
for P in ${PAIRS:-16:8 16:16 16:32 32:32}; do
  TL=${P%%:*}; TU=${P##*:}
  echo "TL=$TL TU=$TU"
  EXG_NARROW_T_L=$TL EXG_NARROW_T_U=$TU EXG_RUN_TIMING=1 timeout 600 python bench.py --steps 3 --warmup 3 --cpu-steps 0 --e2e-steps 1 --profile-steps 1 2>&1 | grep -E "runs\]" | tail -2 | cut -c1-200
done > gpurun_out/sweep_T.log 2>&1
