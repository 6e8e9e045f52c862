mkdir -p gpurun_out
line() { tail -1 $1 | python -c "import json,sys
d=json.loads(sys.stdin.read()); r=d['roofline']; e=d['e2e']
print('$2', 'step_ms', round(d['ms_per_step'],4), 'kernel_ms', round(r.get('kernel_ms',0),4), 'frac', round(r['frac'],3), 'e2e_ms', round(e.get('ms_per_query', 0),4), 'clk', d['clocks']['sm_mhz'], d['clocks']['reasons'])"; }
timeout 900 python -m pytest tests/test_gpu_dense_cut.py tests/test_baseline_sizes.py tests/test_gpu_fullsize.py -q -x -p no:cacheprovider 2>&1 | tail -2
for c in c2 c4; do
  timeout 900 python bench.py --config $c --steps 20 --warmup 5 --no-cpu --no-train > gpurun_out/dc3_${c}.log 2>&1; line gpurun_out/dc3_${c}.log "$c-cut"
  OTF_DENSE_NO_CUT=1 timeout 900 python bench.py --config $c --steps 20 --warmup 5 --no-cpu --no-train > gpurun_out/dc3_${c}_nocut.log 2>&1; line gpurun_out/dc3_${c}_nocut.log "$c-nocut"
done
CFG=c2 bash tools/gpu_dcut_trace.sh 2>&1 | tail -8
