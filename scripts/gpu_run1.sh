#!/bin/bash
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 300 python -m pytest tests/test_gpu.py -q -rA -x -k "umma or tier_a or autograd or zero" 2>&1 | tail -25 > gpurun_out/t_a.log
timeout 240 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1
timeout 300 python bench.py --steps 20 --warmup 5 > gpurun_out/bench_c2.json 2> gpurun_out/bench_c2.err
timeout 300 python bench.py --steps 10 --warmup 3 --config C3 --no-cpu-baseline > gpurun_out/bench_c3.json 2> gpurun_out/bench_c3.err
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_c2.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline --e2e-steps 1 > /dev/null 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:sage_bwd_kernel -s 3 -c 1 -o gpurun_out/prof_bwd_c2 python bench.py --steps 1 --warmup 3 --no-cpu-baseline --e2e-steps 0 > gpurun_out/ncu_bwd.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:sage_fwd_kernel -s 3 -c 1 -o gpurun_out/prof_fwd_c2 python bench.py --steps 1 --warmup 3 --no-cpu-baseline --e2e-steps 0 > gpurun_out/ncu_fwd.log 2>&1
ls gpurun_out
