# full GPU tests, then one bench line per listed config (default: c1 c2 c3 c5a) + top kernels
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/q_tests.log 2>&1; echo tests=$?; tail -2 gpurun_out/q_tests.log
for c in ${CFGS:-c1 c2 c3 c5a}; do
  timeout 600 python bench.py --config $c --steps 20 --warmup 5 --no-cpu > gpurun_out/q_$c.log 2>&1
  tail -1 gpurun_out/q_$c.log | python -c "import json,sys
d=json.loads(sys.stdin.read()); r=d['roofline']
print('$c', round(d['ms_per_step']*1000,1), 'us/step', r['kernel'][:30], round(r['kernel_ms']*1000,1), 'us frac', round(r['frac'],3), 'e2e us', round(d['e2e'].get('ms_per_query')*1000,1), d['clocks']['sm_mhz'], d['clocks']['reasons'])"
  timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/q_launch_$c.csv python bench.py --config $c --steps 5 --warmup 3 --no-cpu > /dev/null 2>&1
  python tools/launches.py gpurun_out/q_launch_$c.csv | grep -E "otf::" | head -4
done
