#!/bin/bash
# K4 ablation sweep for one config (profiling build): prints "<bits> ms_per_step bwd_ms fwd_ms".
cd "$(dirname "$0")/.."
CFG=${CFG:-C2}
for a in ${BITS:-0 1 2 3 4}; do
  SAGE_LIB=$PWD/paper_2603_02170_b200/libsage_trace.so SAGE_ABLATE=$a timeout 200 python bench.py --steps 5 --warmup 3 --config $CFG --no-cpu-baseline --e2e-steps 0 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print($a, d['ms_per_step'], d['roofline']['kernel_ms'], d['roofline']['fwd_kernel_ms'])"
done
