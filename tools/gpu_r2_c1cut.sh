mkdir -p gpurun_out
line() { tail -1 $1 | python -c "import json,sys
d=json.loads(sys.stdin.read()); r=d['roofline']
print('$2', 'step_ms', round(d['ms_per_step'],4), 'kernel_ms', round(r.get('kernel_ms',0),4), 'frac', round(r['frac'],3), 'e2e', round(d['e2e']['ms_per_query'],4), 'clk', d['clocks']['sm_mhz'])"; }
for i in 1 2; do
for v in "" "OTF_DENSE_CUT_D128=1"; do
  env $v timeout 900 python bench.py --config c1 --steps 50 --warmup 5 --no-cpu > gpurun_out/c1c.log 2>&1; line gpurun_out/c1c.log "c1 $v"
done
done
OTF_DENSE_CUT_D128=1 CFG=c1 bash tools/gpu_dcut_trace.sh 2>&1 | tail -8
