mkdir -p gpurun_out
line() { tail -1 $1 | python -c "import json,sys
d=json.loads(sys.stdin.read()); r=d['roofline']
print('$2', 'step_ms', round(d['ms_per_step'],4), 'kernel_ms', round(r.get('kernel_ms',0),4), 'frac', round(r['frac'],3), 'clk', d['clocks']['sm_mhz'])"; }
timeout 900 python -m pytest tests -m gpu -q -x -p no:cacheprovider -k "pq or cut or random or topk or ingest or chunks" > gpurun_out/half_tests.log 2>&1; tail -1 gpurun_out/half_tests.log
for i in 1 2 3; do timeout 900 python bench.py --config c3 --steps 50 --warmup 5 --no-cpu > gpurun_out/half.log 2>&1; line gpurun_out/half.log c3; done
timeout 900 python bench.py --config c3x --steps 20 --warmup 5 --no-cpu > gpurun_out/half.log 2>&1; line gpurun_out/half.log c3x
bash tools/gpu_cut_trace.sh 2>&1 | tail -8
