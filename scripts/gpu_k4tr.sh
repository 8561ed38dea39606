#!/bin/bash
# K4 A/B timelines: trace build of each variant at $CONFIGS (default C4)
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
for v in trace ${TRVARIANTS}; do
  for c in ${TRCONFIGS:-C4}; do
    SAGE_LIB=paper_2603_02170_b200/libsage_$v.so SAGE_ABLATE=8 timeout 300 python scripts/trace_bwd.py $c ${CTA:-0} > gpurun_out/trace_bwd_${v}_$c.txt 2>&1
    echo "$v $c $(tail -1 gpurun_out/trace_bwd_${v}_$c.txt)"
  done
done
