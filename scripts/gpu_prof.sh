#!/bin/bash
# ncu evidence for one config: launch list (cold, serialised) + one --set full capture of a kernel.
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
CFG=${CFG:-C2}; K=${K:-sage_bwd_kernel}; TAG=${TAG:-x}
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_${TAG}_${CFG}.csv python bench.py --config $CFG --steps 2 --warmup 3 --no-cpu-baseline --e2e-steps 0 > /dev/null 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:$K -s 3 -c 1 -o gpurun_out/prof_${TAG}_${CFG}_$K -f python bench.py --config $CFG --steps 1 --warmup 3 --no-cpu-baseline --e2e-steps 0 > gpurun_out/ncu_${TAG}.log 2>&1
ls -la gpurun_out
