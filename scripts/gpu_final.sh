#!/bin/bash
# Round-end evidence in one GPU call (TAG names the files): GPU tests, smoke, the default bench line (C4 with
# cpu_baseline and in-run parity), the reference arm at the driver's default steps, C2/C3/C5 lines, variant
# lines, the 1K-32K sweep, launch lists and ncu --set full captures of K4 / K2 / K1 at C4 (summaries only).
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
TAG=${TAG:-final}
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,driver_version --format=csv > gpurun_out/gpu_info_$TAG.txt 2>&1
if [ -z "$NO_TESTS" ]; then
  timeout 1500 python -m pytest tests/ -m gpu -q -rA > gpurun_out/t_gpu_$TAG.log 2>&1; echo "pytest exit $?" >> gpurun_out/t_gpu_$TAG.log
  tail -2 gpurun_out/t_gpu_$TAG.log
  timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_$TAG.log 2>&1; tail -1 gpurun_out/smoke_$TAG.log
fi
( time timeout 900 python bench.py ) > gpurun_out/bench_${TAG}_default.json 2> gpurun_out/bench_${TAG}_default.err
( time timeout 1500 python bench.py --impl reference ) > gpurun_out/bench_${TAG}_ref.json 2> gpurun_out/bench_${TAG}_ref.err
for c in C2 C3 C5; do
  timeout 600 python bench.py --config $c --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/bench_${TAG}_$c.json 2> gpurun_out/bench_${TAG}_$c.err
done
for a in --pv-fp8 --p-u8 --deterministic --fine-bwd; do
  timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline $a > gpurun_out/bench_${TAG}_C4${a//-/_}.json 2> /dev/null
done
timeout 600 python bench.py --config C5 --steps 10 --warmup 3 --no-cpu-baseline --qk-norm > gpurun_out/bench_${TAG}_C5_qk_norm.json 2> /dev/null
TAG=$TAG bash scripts/gpu_sweep.sh > gpurun_out/sweep_$TAG.txt 2>&1
for CFG in C4 C3 C2; do
  timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_${TAG}_${CFG}.csv \
    python bench.py --config $CFG --steps 2 --warmup 3 --no-cpu-baseline --no-parity --e2e-steps 0 > /dev/null 2>&1
done
for K in sage_bwd_kernel sage_fwd_kernel quantize_kernel; do
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:$K -s 2 -c 1 \
    -o gpurun_out/prof_${TAG}_C4_$K -f python bench.py --config C4 --steps 1 --warmup 3 --no-cpu-baseline --no-parity --e2e-steps 0 > /dev/null 2>&1
done
cp profiles/ncu_summary.json gpurun_out/ncu_summary_$TAG.json
python scripts/ncu_summary.py json gpurun_out/ncu_summary_$TAG.json gpurun_out/prof_${TAG}_*.ncu-rep > /dev/null 2>&1
for f in gpurun_out/prof_${TAG}_*.ncu-rep; do python scripts/ncu_summary.py rep $f; done > gpurun_out/ncu_$TAG.txt 2>&1
python scripts/ncu_lines.py gpurun_out/prof_${TAG}_C4_sage_bwd_kernel.ncu-rep 40 > gpurun_out/ncu_lines_${TAG}_k4.txt 2>&1
rm -f gpurun_out/prof_${TAG}_*.ncu-rep
cat gpurun_out/sweep_$TAG.txt
tail -c 300 gpurun_out/bench_${TAG}_default.err gpurun_out/bench_${TAG}_ref.err
