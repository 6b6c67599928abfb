# one-call sweep of plan knobs at 1M with a shared factor cache:
# prints "<env> -> value" per variant (bench.py default steps)
export EXG_FACTOR_CACHE=/tmp/exg_fc
mkdir -p gpurun_out
for V in ${VARIANTS:-"X=0" "EXG_ABSORB_ROWS=4096" "EXG_ABSORB_ROWS=16384" "EXG_ABSORB_ROWS=32768" "EXG_LEVELS=asap" "EXG_LEVELS=alap" "EXG_CHAIN_OLD=6" "EXG_CHAIN_SPIN=200" "X=1"}; do
  v=$(env $V timeout 240 python bench.py --cpu-steps 0 2>/dev/null | tail -1 | python -c "import sys,json; d=json.loads(sys.stdin.read()); print(d['value'], d['e2e']['value'])" 2>&1)
  echo "$V -> $v"
done > gpurun_out/sweep_knobs.log 2>&1
