#!/bin/bash
# The metric's sequence-length sweep (S1K..S32K: B = 32768/N, H = 32, d = 128, causal): one bench line each.
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
for c in S1K S2K S4K S8K S16K S32K; do
  timeout 600 python bench.py --config $c --steps 10 --warmup 3 --no-cpu-baseline --e2e-steps 2 > gpurun_out/sweep_${TAG:-x}_$c.json 2> gpurun_out/sweep_${TAG:-x}_$c.err
done
for c in S1K S2K S4K S8K S16K S32K; do
  python -c "import json; d=json.load(open('gpurun_out/sweep_${TAG:-x}_$c.json')); r=d['roofline']; print('$c', round(d['value'],1), round(d['ms_per_step'],3), round(r['kernel_ms'],3), round(r['fwd_kernel_ms'],3), round(r['frac'],3), round(d['e2e']['value'],1))" 2>&1 | tail -1
done
