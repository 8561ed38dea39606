#!/bin/bash
# The round's bench lines: default run (C2 + cpu_baseline), the reference arm, and C3-C5.
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
TAG=${TAG:-r01}
timeout 600 python bench.py > gpurun_out/bench_${TAG}_C2.json 2> gpurun_out/bench_${TAG}_C2.err
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/bench_${TAG}_ref.json 2> gpurun_out/bench_${TAG}_ref.err
for c in ${CONFIGS:-C3 C4 C5}; do
  timeout 900 python bench.py --config $c --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/bench_${TAG}_$c.json 2> gpurun_out/bench_${TAG}_$c.err
done
tail -c 400 gpurun_out/bench_${TAG}_*.err
