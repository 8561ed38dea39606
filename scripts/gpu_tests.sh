#!/bin/bash
# Run the GPU test tiers with hard timeouts (a hung kernel must not hang the box).
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/gpu_info.txt 2>&1
timeout 300 python -m pytest tests/test_gpu.py -x -q -k "umma" 2>&1 | tail -30 > gpurun_out/t_umma.log
timeout 600 python -m pytest tests/test_gpu.py -q -k "not umma" ${PYTEST_EXTRA} 2>&1 | tail -60 > gpurun_out/t_parity.log
tail -5 gpurun_out/t_umma.log gpurun_out/t_parity.log
