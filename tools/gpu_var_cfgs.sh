# A/B every tools/var/*.so on the configs in CFGS (step, scoring kernel, launch list of the top kernels)
mkdir -p gpurun_out
cp paper_1407_4764_b200/libotf_b200.so /tmp/otf_default.so
for round in 1 2; do
for v in tools/var/*.so; do
  cp $v paper_1407_4764_b200/libotf_b200.so
  for c in ${CFGS:-c3}; do
    timeout -k 10 300 python bench.py --config $c --steps 50 --warmup 5 --no-cpu > gpurun_out/var.log 2>&1
    echo var=$(basename $v) $c $(tail -1 gpurun_out/var.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['ms_per_step']*1000,1), 'us/step scan', round(d['roofline']['kernel_ms']*1000,1), 'e2e', round(d['e2e']['ms_per_query']*1000,1), d['clocks']['sm_mhz'])" 2>&1 | tail -1)
  done
done
done
for v in tools/var/*.so; do
  cp $v paper_1407_4764_b200/libotf_b200.so
  for c in ${CFGS:-c3}; do
    timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/varl.csv python bench.py --config $c --steps 5 --warmup 3 --no-cpu > /dev/null 2>&1
    echo "launches var=$(basename $v) $c"; python tools/launches.py gpurun_out/varl.csv | grep -E "otf::" | head -4 | cut -c1-110
  done
done
cp /tmp/otf_default.so paper_1407_4764_b200/libotf_b200.so
