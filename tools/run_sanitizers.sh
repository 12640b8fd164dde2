#!/bin/bash
# compute-sanitizer over tools/sanitize_workload.py (run on the GPU box). Logs -> gpurun_out/sanitize_*.log
cd "$(dirname "$0")/.."
for tool in memcheck racecheck synccheck initcheck; do
  extra=""
  [ "$tool" = "memcheck" ] && extra="--leak-check full"
  timeout 1500 compute-sanitizer --tool $tool $extra --target-processes all --print-limit 50 \
    python tools/sanitize_workload.py > gpurun_out/sanitize_$tool.log 2>&1
  echo "exit=$?" >> gpurun_out/sanitize_$tool.log
done
