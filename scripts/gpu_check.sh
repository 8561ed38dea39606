#!/bin/bash
# Fast correctness probe of the built libraries (check_variants.py) then bench lines for $CONFIGS.
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
TAG=${TAG:-x}
CUDA_LAUNCH_BLOCKING=1 timeout 300 python scripts/check_variants.py > gpurun_out/check_$TAG.log 2>&1; echo "check exit $?" >> gpurun_out/check_$TAG.log
cat gpurun_out/check_$TAG.log
NO_TESTS=1 TAG=$TAG bash scripts/gpu_quick.sh
