#!/bin/bash
# compute-sanitizer (memcheck, racecheck, synccheck) over tools/sanitize_case.py
mkdir -p gpurun_out
timeout 300 python tools/sanitize_case.py > gpurun_out/sanitize_plain.log 2>&1; echo "plain rc=$?"
for tool in memcheck racecheck synccheck; do
  timeout ${SAN_TIMEOUT:-1500} compute-sanitizer --tool $tool --error-exitcode 9 python tools/sanitize_case.py > gpurun_out/sanitize_$tool.log 2>&1
  echo "$tool rc=$?"; tail -4 gpurun_out/sanitize_$tool.log
done
