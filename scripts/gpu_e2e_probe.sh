cd /root/repo
for ch in 16 32 64; do
  timeout 600 python bench.py --config C4 --steps 5 --warmup 3 --no-cpu-baseline --no-parity --e2e-steps 3 --e2e-chunks $ch > gpurun_out/e2e_$ch.json 2>/dev/null
  python -c "import json; d=json.load(open('gpurun_out/e2e_$ch.json')); print('chunks $ch', round(d['value'],1), 'e2e', round(d['e2e']['value'],1), round(d['e2e']['ms_per_step'],2))"
done
SAGE_ABLATE=8 timeout 300 python scripts/trace_bwd.py C4 0 > gpurun_out/trace_bwd_prod_C4.txt 2>&1; tail -1 gpurun_out/trace_bwd_prod_C4.txt
