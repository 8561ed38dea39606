#!/bin/bash
# ragged-N tests, then bench lines twice per config (noise check)
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_ragged.py -x -q > gpurun_out/t_rag.log 2>&1; echo "ragged tests exit $?: $(tail -1 gpurun_out/t_rag.log)"
for rep in 1 2; do
for c in ${CONFIGS:-C4 C3 C2}; do
  timeout 600 python bench.py --config $c --steps 10 --warmup 3 --no-cpu-baseline --e2e-steps 0 > gpurun_out/bench_rag_$c.json 2> gpurun_out/bench_rag_$c.err
  python -c "import json; d=json.load(open('gpurun_out/bench_rag_$c.json')); r=d['roofline']; print('$c', round(d['value'],1), 'K4', round(r['kernel_ms'],4), 'K2', round(r['fwd_kernel_ms'],4), 'parity', d.get('parity',{}).get('ok'))" || tail -5 gpurun_out/bench_rag_$c.err
done
done
