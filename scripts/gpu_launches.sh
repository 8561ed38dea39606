#!/bin/bash
# ncu launch lists (cold, serialised per-kernel durations) of one bench step: CONFIGS x ARGS variants.
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
for c in ${CONFIGS:-C5}; do
  timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_${TAG:-x}_$c.csv python bench.py --config $c --steps 1 --warmup 3 --no-cpu-baseline --e2e-steps 0 $ARGS > /dev/null 2>&1
done
python scripts/launch_table.py gpurun_out/launches_${TAG:-x}_*.csv
