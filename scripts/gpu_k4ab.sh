#!/bin/bash
# K4 A/B: correctness probe of each build, d=128 GPU parity + fused-tile tests, then variant bench lines.
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
out=gpurun_out/k4ab.txt; : > $out
for v in prod ${VARIANTS}; do
  lib=paper_2603_02170_b200/libsage.so; [ $v != prod ] && lib=paper_2603_02170_b200/libsage_$v.so
  SAGE_LIB=$lib timeout 300 python scripts/check_variants.py >> $out 2>&1
done
timeout 900 python -m pytest tests/test_gpu.py tests/test_gpu_tiles.py -x -q > gpurun_out/t_k4ab.log 2>&1
echo "tests exit $?: $(tail -1 gpurun_out/t_k4ab.log)" >> $out
VARIANTS="$VARIANTS" CONFIGS="${CONFIGS:-C4 C3 C5}" bash scripts/gpu_variants.sh > /dev/null 2>&1
cat gpurun_out/variants.txt >> $out
cat $out
