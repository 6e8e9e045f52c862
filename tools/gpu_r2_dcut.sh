# dense cut path: its tests, the dense parity tests, then C1 / C2 / C3 / C4 bench lines (new L2 flush)
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_dense_cut.py -q -x -p no:cacheprovider > gpurun_out/dc_tests.log 2>&1; echo dcut_tests=$?; tail -15 gpurun_out/dc_tests.log
timeout 900 python -m pytest tests -m gpu -q -x -p no:cacheprovider -k "dense or baseline or fullsize or session or sharded or graph" > gpurun_out/dc_tests2.log 2>&1; echo dense_tests=$?; tail -3 gpurun_out/dc_tests2.log
for c in c1 c2 c3 c4; do
  timeout 900 python bench.py --config $c --steps 30 --warmup 5 --no-cpu > gpurun_out/dc_$c.log 2>&1
  tail -1 gpurun_out/dc_$c.log | python -c "import json,sys
d=json.loads(sys.stdin.read()); r=d['roofline']
print('$c', round(d['ms_per_step']*1000,1), 'us/step kernel', round(r['kernel_ms']*1000,1), 'us frac', round(r['frac'],3), 'e2e us', round(d['e2e']['ms_per_query']*1000,1), d['clocks']['sm_mhz'], d['clocks']['reasons'], 'launches', d['gpu_launches'])"
done
OTF_DENSE_NO_CUT=1 timeout 900 python bench.py --config c1 --steps 30 --warmup 5 --no-cpu > gpurun_out/dc_c1_nocut.log 2>&1
tail -1 gpurun_out/dc_c1_nocut.log | python -c "import json,sys
d=json.loads(sys.stdin.read()); r=d['roofline']
print('c1 nocut', round(d['ms_per_step']*1000,1), 'us/step kernel', round(r['kernel_ms']*1000,1), 'us frac', round(r['frac'],3), 'e2e us', round(d['e2e']['ms_per_query']*1000,1))"
