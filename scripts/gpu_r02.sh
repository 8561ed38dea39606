#!/bin/bash
# Round-2 GPU pass: GPU tests (incl. the fused-tile parity), smoke, the default bench line (C4 + parity +
# cpu_baseline), the reference arm, C2/C3 lines, and the C4 launch list.  TAG names the outputs.
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
TAG=${TAG:-r02a}
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,driver_version --format=csv > gpurun_out/gpu_info_$TAG.txt 2>&1
timeout ${TEST_TIMEOUT:-1500} python -m pytest tests/ -m gpu -q -rA ${PYTEST_K:+-k "$PYTEST_K"} > gpurun_out/t_gpu_$TAG.log 2>&1
echo "pytest exit $?" >> gpurun_out/t_gpu_$TAG.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_$TAG.log 2>&1
timeout 900 python bench.py > gpurun_out/bench_${TAG}_C4.json 2> gpurun_out/bench_${TAG}_C4.err
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/bench_${TAG}_ref.json 2> gpurun_out/bench_${TAG}_ref.err
for c in ${CONFIGS:-C2 C3}; do
  timeout 600 python bench.py --config $c --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/bench_${TAG}_$c.json 2> gpurun_out/bench_${TAG}_$c.err
done
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_${TAG}_C4.csv \
  python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-parity --e2e-steps 0 > /dev/null 2>&1
tail -3 gpurun_out/t_gpu_$TAG.log
tail -c 300 gpurun_out/bench_${TAG}_*.err
