cd /root/repo; mkdir -p gpurun_out
SAGE_DEBUG=1 timeout 120 python -m pytest tests/test_gpu.py -x -q -k autograd 2>&1 | grep -E "libsage|passed|failed" > gpurun_out/t_ag.log
for a in 0 1 2 3 4; do
  SAGE_LIB=$PWD/paper_2603_02170_b200/libsage_trace.so SAGE_ABLATE=$a timeout 200 python bench.py --steps 10 --warmup 3 --config C2 --no-cpu-baseline --e2e-steps 0 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print($a, d['ms_per_step'], d['roofline']['kernel_ms'], d['roofline']['fwd_kernel_ms'])" >> gpurun_out/abl.txt
done
SAGE_ABLATE=0 timeout 200 python bench.py --steps 10 --warmup 3 --config C3 --no-cpu-baseline --e2e-steps 0 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('C3', d['ms_per_step'], d['roofline']['kernel_ms'], d['roofline']['fwd_kernel_ms'])" >> gpurun_out/abl.txt
