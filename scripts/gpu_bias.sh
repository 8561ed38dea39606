#!/bin/bash
# Q-smoothing bias: correctness (check_variants, the Q-smoothing GPU tests) and the C3 A/B of the tensor-core
# bias kernel against the CUDA-core one (libsage_biascuda.so), with a launch list of C3.
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
TAG=${TAG:-x}
CUDA_LAUNCH_BLOCKING=1 timeout 300 python scripts/check_variants.py > gpurun_out/check_$TAG.log 2>&1; echo "check exit $?" >> gpurun_out/check_$TAG.log
cat gpurun_out/check_$TAG.log
timeout 900 python -m pytest tests/test_gpu.py -q -x -k "tier_a or outlier_kq or qs or q_smooth" > gpurun_out/t_bias_$TAG.log 2>&1; tail -2 gpurun_out/t_bias_$TAG.log
CONFIGS="C3" VARIANTS="biascuda" bash scripts/gpu_variants.sh
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_${TAG}_C3.csv \
  python bench.py --config C3 --steps 2 --warmup 3 --no-cpu-baseline --no-parity --e2e-steps 0 > /dev/null 2>&1
python scripts/launch_table.py gpurun_out/launches_${TAG}_C3.csv
