#!/bin/bash
# ncu evidence for the round's profiles/: per config a cold launch list and one --set full
# capture of each fused kernel (K4 bwd, K2 fwd) and the quantiser (K1).  One GPU, short benches.
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
TAG=${TAG:-r01}
for CFG in ${CONFIGS:-C2 C3}; do
  timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file gpurun_out/launches_${TAG}_${CFG}.csv \
    python bench.py --config $CFG --steps 2 --warmup 3 --no-cpu-baseline --e2e-steps 0 > /dev/null 2>&1
  for K in sage_bwd_kernel sage_fwd_kernel quantize_kernel ${EXTRA_K}; do
    timeout 600 ncu --set full --clock-control none --import-source on -k regex:$K -s 2 -c 1 \
      -o gpurun_out/prof_${TAG}_${CFG}_${K} -f \
      python bench.py --config $CFG --steps 1 --warmup 3 --no-cpu-baseline --e2e-steps 0 > /dev/null 2>&1
  done
done
ls -la gpurun_out
