#!/bin/bash
# One build->measure iteration on the GPU box: parity tests, then short benches.
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/gpu_info.txt 2>&1
timeout 420 python -m pytest tests/test_gpu.py -x -q -k "${TESTK:-not full_size}" 2>&1 | tail -30 > gpurun_out/t_parity.log
echo "parity exit $?" >> gpurun_out/t_parity.log
for c in ${CONFIGS:-C2 C3}; do
  timeout 300 python bench.py --steps 10 --warmup 3 --config $c --no-cpu-baseline --e2e-steps 1 > gpurun_out/bench_$c.json 2> gpurun_out/bench_$c.err
done
tail -3 gpurun_out/t_parity.log; cat gpurun_out/bench_*.json
