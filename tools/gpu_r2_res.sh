mkdir -p gpurun_out
line() { tail -1 $1 | python -c "import json,sys
d=json.loads(sys.stdin.read()); r=d['roofline']; t=d.get('training') or {}
print('$2', 'step_ms', round(d['ms_per_step'],4), 'kernel_ms', round(r.get('kernel_ms',0),4), 'frac', round(r['frac'],3), 'trainer/s', round(t.get('trainer_steps_per_s',0)), 'clk', d['clocks']['sm_mhz'], d['clocks']['reasons'])"; }
for i in 1 2; do
for v in 0 1 2; do
  OTF_BENCH_RESERVE_SMS=$v timeout 900 python bench.py --config c4 --steps 30 --warmup 5 --no-cpu > gpurun_out/res.log 2>&1; line gpurun_out/res.log "c4 reserve=$v"
done
done
