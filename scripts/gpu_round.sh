#!/bin/bash
# Round evidence in one GPU call: full GPU test suite, fidelity report, bench lines (C2 default + cpu
# baseline, reference arm, C3-C5, C5 with --qk-norm / --p-u8), ncu launch lists + full captures.
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
TAG=${TAG:-r01}
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,driver_version --format=csv > gpurun_out/gpu_info.txt 2>&1
timeout 900 python -m pytest tests/ -m gpu -q -rA 2>&1 | tail -80 > gpurun_out/t_gpu_all.log
TAG=$TAG CONFIGS="C3 C4 C5" bash scripts/gpu_bench_all.sh > /dev/null 2>&1
for a in --qk-norm --p-u8 --fine-bwd --deterministic; do
  timeout 600 python bench.py --config C5 --steps 10 --warmup 3 --no-cpu-baseline $a > gpurun_out/bench_${TAG}_C5${a//-/_}.json 2> /dev/null
done
TAG=$TAG CONFIGS="${NCU_CONFIGS:-C2 C3 C4}" EXTRA_K="${EXTRA_K}" bash scripts/gpu_evidence.sh > /dev/null 2>&1
ls gpurun_out
# summaries here (the .ncu-rep files are too large to bring back: gpurun_out is capped at 64 MiB)
python scripts/ncu_summary.py json gpurun_out/ncu_summary_$TAG.json gpurun_out/prof_*.ncu-rep > /dev/null 2>&1
for f in gpurun_out/prof_*.ncu-rep; do python scripts/ncu_summary.py rep $f; done > gpurun_out/ncu_$TAG.txt 2>&1
ls -la gpurun_out/prof_*.ncu-rep > gpurun_out/ncu_reports_$TAG.txt
rm -f gpurun_out/prof_*.ncu-rep
du -sh gpurun_out
