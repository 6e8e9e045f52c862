mkdir -p gpurun_out
line() { tail -1 $1 | python -c "import json,sys
d=json.loads(sys.stdin.read()); r=d['roofline']
print('$2', 'step_ms', round(d['ms_per_step'],4), 'kernel_ms', round(r.get('kernel_ms',0),4), 'frac', round(r['frac'],3), 'e2e', round(d['e2e']['ms_per_query'],4), 'clk', d['clocks']['sm_mhz'], d['clocks']['reasons'])"; }
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_topk_chunks.py tests/test_gpu_fullsize.py tests/test_baseline_sizes.py -q -x -p no:cacheprovider 2>&1 | tail -2
for i in 1 2; do
for v in "" "OTF_DENSE_STATIC=1"; do
  env $v timeout 900 python bench.py --config c1 --steps 50 --warmup 5 --no-cpu > gpurun_out/c1v.log 2>&1; line gpurun_out/c1v.log "c1 $v"
  env $v OTF_DENSE_NO_CUT=1 timeout 900 python bench.py --config c2 --steps 20 --warmup 5 --no-cpu > gpurun_out/c1v.log 2>&1; line gpurun_out/c1v.log "c2-nocut $v"
done
done
