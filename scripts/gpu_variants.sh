#!/bin/bash
# Profiling A/B: bench the production lib and each libsage_<VARIANT>.so (build.build_variant) on CONFIGS,
# optionally after the GPU parity tests (TESTS=1).
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
out=gpurun_out/variants.txt; : > $out
if [ -n "$TESTS" ]; then
  timeout 420 python -m pytest tests/test_gpu.py -x -q -k "${TESTK:-not full_size}" > gpurun_out/t_parity.log 2>&1
  echo "parity exit $?: $(tail -1 gpurun_out/t_parity.log)" >> $out
fi
for v in prod ${VARIANTS}; do
  lib=paper_2603_02170_b200/libsage.so; [ $v != prod ] && lib=paper_2603_02170_b200/libsage_$v.so
  for c in ${CONFIGS:-C2}; do
    SAGE_LIB=$lib timeout 300 python bench.py --steps 10 --warmup 3 --config $c --no-cpu-baseline --e2e-steps 0 > gpurun_out/var.json 2>gpurun_out/var.err
    python -c "import json; d=json.load(open('gpurun_out/var.json')); r=d['roofline']; print('$v $c', round(d['value'],1), 'K4', round(r['kernel_ms'],4), 'K2', round(r['fwd_kernel_ms'],4))" >> $out 2>&1 || tail -3 gpurun_out/var.err >> $out
  done
done
cat $out
