mkdir -p gpurun_out
line() { tail -1 $1 | python -c "import json,sys
d=json.loads(sys.stdin.read()); r=d['roofline']
print('$2', 'step_ms', round(d['ms_per_step'],4), 'kernel_ms', round(r.get('kernel_ms',0),4), 'frac', round(r['frac'],3), 'e2e', round(d['e2e']['ms_per_query'],4), 'clk', d['clocks']['sm_mhz'], d['clocks']['reasons'])"; }
timeout 900 python -m pytest tests -m gpu -q -x -p no:cacheprovider -k "parity or topk or fullsize or baseline or graph or session" 2>&1 | tail -2
for i in 1 2; do
for v in "" "OTF_TOPK_NO_PDL=1"; do
  env $v timeout 900 python bench.py --config c1 --steps 50 --warmup 5 --no-cpu > gpurun_out/pv.log 2>&1; line gpurun_out/pv.log "c1 $v"
done
done
for v in "" "OTF_TOPK_NO_PDL=1"; do
  env $v timeout 900 python bench.py --config c5a --steps 10 --warmup 3 --no-cpu > gpurun_out/pv.log 2>&1; line gpurun_out/pv.log "c5a $v"
done
