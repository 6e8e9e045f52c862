mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -q -x -p no:cacheprovider -k "pq or cut or c3 or quantized or random or topk or session" > gpurun_out/pq_tests.log 2>&1; echo pq_tests=$?; tail -15 gpurun_out/pq_tests.log
for v in "" ; do
  env $v timeout 900 python bench.py --config c3 --steps 50 --warmup 5 --no-cpu > gpurun_out/pq_c3.log 2>&1
  tail -1 gpurun_out/pq_c3.log | python -c "import json,sys
d=json.loads(sys.stdin.read()); r=d['roofline']
print('c3 $v', round(d['ms_per_step']*1000,1), 'us/step kernel', round(r['kernel_ms']*1000,1), 'us frac', round(r['frac'],3), 'e2e us', round(d['e2e']['ms_per_query']*1000,1), d['clocks']['sm_mhz'], d['clocks']['reasons'])"
done
bash tools/gpu_cut_trace.sh
