#!/bin/bash
# Iteration pass: GPU tests (PYTEST_K filter optional), then bench lines for $CONFIGS (no cpu baseline).
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
TAG=${TAG:-x}
if [ -z "$NO_TESTS" ]; then
  timeout ${TEST_TIMEOUT:-1200} python -m pytest tests/ -m gpu -x -q ${PYTEST_K:+-k "$PYTEST_K"} > gpurun_out/t_gpu_$TAG.log 2>&1
  echo "pytest exit $?" >> gpurun_out/t_gpu_$TAG.log
  tail -3 gpurun_out/t_gpu_$TAG.log
fi
for c in ${CONFIGS:-C4 C3 C2}; do
  timeout 600 python bench.py --config $c --steps 10 --warmup 3 --no-cpu-baseline --e2e-steps 0 ${BENCH_ARGS} > gpurun_out/bench_${TAG}_$c.json 2> gpurun_out/bench_${TAG}_$c.err
  python -c "import json; d=json.load(open('gpurun_out/bench_${TAG}_$c.json')); r=d['roofline']; print('$c', round(d['value'],1), 'K4', round(r['kernel_ms'],4), 'K2', round(r['fwd_kernel_ms'],4), 'parity', d.get('parity',{}).get('ok'), d['clocks']['reasons'])" || tail -5 gpurun_out/bench_${TAG}_$c.err
done
