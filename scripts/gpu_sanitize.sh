#!/bin/bash
# compute-sanitizer passes, one tool at a time (each capped); logs to gpurun_out/sanitize_<tool>_<TAG>.log
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
TAG=${TAG:-x}
for tool in ${TOOLS:-racecheck synccheck memcheck}; do
  timeout ${SAN_TIMEOUT:-900} compute-sanitizer --tool $tool --print-limit 50 python scripts/sanitize_run.py \
    > gpurun_out/sanitize_${tool}_$TAG.log 2>&1
  echo "exit $?" >> gpurun_out/sanitize_${tool}_$TAG.log
  tail -4 gpurun_out/sanitize_${tool}_$TAG.log
done
