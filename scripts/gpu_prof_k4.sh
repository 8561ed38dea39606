#!/bin/bash
# K4 evidence at one config: clock64 timeline (trace build) + one ncu --set full capture with source,
# summarised here (per-line stalls) so only text comes back.
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
CFG=${CFG:-C4}; TAG=${TAG:-x}; K=${K:-sage_bwd_kernel}
SAGE_ABLATE=8 timeout 300 python scripts/trace_bwd.py $CFG 0 > gpurun_out/trace_bwd_${TAG}_$CFG.txt 2>&1
SAGE_ABLATE=8 TRACE_FWD=1 timeout 300 python scripts/trace_bwd.py $CFG 0 > gpurun_out/trace_fwd_${TAG}_$CFG.txt 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:$K -s 3 -c 1 \
  -o gpurun_out/prof_${TAG}_${CFG} -f python bench.py --config $CFG --steps 1 --warmup 3 --no-cpu-baseline \
  --no-parity --e2e-steps 0 > gpurun_out/ncu_${TAG}.log 2>&1
python scripts/ncu_lines.py gpurun_out/prof_${TAG}_${CFG}.ncu-rep 60 > gpurun_out/ncu_lines_${TAG}_$CFG.txt 2>&1
python scripts/ncu_summary.py rep gpurun_out/prof_${TAG}_${CFG}.ncu-rep > gpurun_out/ncu_sum_${TAG}_$CFG.txt 2>&1
ncu -i gpurun_out/prof_${TAG}_${CFG}.ncu-rep --page raw --csv > gpurun_out/ncu_raw_${TAG}_$CFG.csv 2>&1
rm -f gpurun_out/prof_${TAG}_${CFG}.ncu-rep
ls -la gpurun_out | tail -5
