# A/B of the run timing between the default library and exp variants
export EXG_FACTOR_CACHE=/tmp/exg_fc
mkdir -p gpurun_out
for V in default ${VARIANTS:-}; do
  if [ "$V" = default ]; then unset EXG_LIB; else export EXG_LIB=exp/$V/libexg.so; fi
  echo "variant $V"
  EXG_RUN_TIMING=1 timeout 600 python bench.py --steps 3 --warmup 3 --cpu-steps 0 --profile-steps 1 2>&1 | grep -E "runs\]|metric" | tail -3 | cut -c1-160
done > gpurun_out/ab.log 2>&1
