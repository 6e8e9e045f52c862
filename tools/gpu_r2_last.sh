# Last round-2 refresh after the selection-prologue change: tests, smoke, bench lines, and the
# launch lists + one --set full capture for the two changed rank kernels (C1, C3).
mkdir -p gpurun_out
line() { tail -1 $1 | python -c "import json,sys
d=json.loads(sys.stdin.read()); r=d['roofline']; e=d['e2e']
print('$2', 'step_ms', round(d['ms_per_step'],4), 'value', '%.4g' % d['value'], 'kernel_ms', round(r.get('kernel_ms',0),4), 'frac', round(r['frac'],3) if r.get('frac') else None, 'e2e_ms', round(e.get('ms_per_query', 0),4), 'clk', d['clocks']['sm_mhz'], d['clocks']['reasons'], 'launches', d['gpu_launches'])"; }
timeout 2400 python -m pytest tests -m gpu -q -x -p no:cacheprovider > gpurun_out/r2f_tests.log 2>&1; echo tests=$?; tail -1 gpurun_out/r2f_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" 2>&1 | tail -1
timeout 900 python bench.py > gpurun_out/r2f_bench.log 2>&1; echo bench=$?; line gpurun_out/r2f_bench.log default
for c in c1 c2 c3 c3x c4; do
  timeout 900 python bench.py --config $c --steps 20 --warmup 5 --no-cpu > gpurun_out/r2f_$c.log 2>&1; line gpurun_out/r2f_$c.log $c
done
for spec in "c1:dense_rank_cut:1" "c3:pq_rank_cut|pq_build_lut:2"; do
  IFS=: read cfg kr cnt <<< "$spec"
  timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_r2f_$cfg.csv \
      python bench.py --config $cfg --steps 5 --warmup 3 --no-cpu --no-train > /dev/null 2>&1; echo launches_$cfg=$?
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:"$kr" -s 4 -c $cnt -o gpurun_out/prof_r2f_$cfg \
      python bench.py --config $cfg --steps 3 --warmup 3 --no-cpu --no-train > /dev/null 2>&1; echo full_$cfg=$?
done
timeout 600 python tools/latency_probe.py c1 c3 c2 > gpurun_out/r2f_lat.log 2>&1; tail -12 gpurun_out/r2f_lat.log
