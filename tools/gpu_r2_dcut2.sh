mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_dense_cut.py -q -x -p no:cacheprovider > gpurun_out/dc_tests.log 2>&1; echo dcut_tests=$?; tail -3 gpurun_out/dc_tests.log
for c in c1 c2; do
  timeout 900 python bench.py --config $c --steps 30 --warmup 5 --no-cpu > gpurun_out/dc_$c.log 2>&1
  tail -1 gpurun_out/dc_$c.log | python -c "import json,sys
d=json.loads(sys.stdin.read()); r=d['roofline']
print('$c', round(d['ms_per_step']*1000,1), 'us/step kernel', round(r['kernel_ms']*1000,1), 'us frac', round(r['frac'],3), 'e2e us', round(d['e2e']['ms_per_query']*1000,1), d['clocks']['sm_mhz'], d['clocks']['reasons'], 'launches', d['gpu_launches'])"
done
bash tools/gpu_dcut_trace.sh
for c in c1 c2; do
  OTF_DENSE_NO_CUT=1 timeout 900 python bench.py --config $c --steps 30 --warmup 5 --no-cpu > gpurun_out/dc_${c}_nocut.log 2>&1
  tail -1 gpurun_out/dc_${c}_nocut.log | python -c "import json,sys
d=json.loads(sys.stdin.read()); r=d['roofline']
print('$c nocut', round(d['ms_per_step']*1000,1), 'us/step kernel', round(r['kernel_ms']*1000,1), 'us frac', round(r['frac'],3), 'e2e us', round(d['e2e']['ms_per_query']*1000,1))"
done
