#!/bin/bash
# K4 / K2 clock64 timelines (libsage_trace.so, SAGE_ABLATE bit 8) for the configs in $CONFIGS.
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
for c in ${CONFIGS:-C4}; do
  SAGE_ABLATE=8 timeout 300 python scripts/trace_bwd.py $c ${CTA:-0} > gpurun_out/trace_bwd_$c.txt 2>&1
  SAGE_ABLATE=8 TRACE_FWD=1 timeout 300 python scripts/trace_bwd.py $c ${CTA:-0} > gpurun_out/trace_fwd_$c.txt 2>&1
done
