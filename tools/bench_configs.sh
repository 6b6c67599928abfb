# per-config transient throughput, one process per config with its own time limit
mkdir -p gpurun_out
: > gpurun_out/configs.jsonl
for spec in ${SPECS:-0:300 3:300 2:900 4:900 1:900}; do
  c=${spec%%:*}; lim=${spec##*:}
  echo "== config $c (limit ${lim}s)" >> gpurun_out/configs.log
  timeout $lim python tools/bench_configs.py --configs $c --cpu-seconds ${CPU_S:-20} --out gpurun_out/configs_c$c.json \
      >> gpurun_out/configs.jsonl 2>> gpurun_out/configs.log
  echo "rc=$?" >> gpurun_out/configs.log
done
