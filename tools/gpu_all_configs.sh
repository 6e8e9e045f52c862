# One bench line per config (no CPU leg except the default), for the DESIGN.md table.
mkdir -p gpurun_out
for c in c1 c2 c3 c4 c5a c5b c3e c3k; do
  timeout 900 python bench.py --config $c --steps 10 --warmup 3 --no-cpu > gpurun_out/all_$c.log 2>&1
  tail -1 gpurun_out/all_$c.log | python -c "import json,sys
d=json.loads(sys.stdin.read()); r=d['roofline']
print('$c', round(d['value']/1e9,3), 'G/s', round(d['ms_per_step'],4), 'ms', r['kernel'][:40], round(r['kernel_ms'],4), 'ms frac', round(r['frac'],3), 'e2e ms', round(d['e2e'].get('ms_per_query', d['e2e']['value']),3), d['clocks']['sm_mhz'], d['clocks']['reasons'], 'launches', d['gpu_launches'])"
done
