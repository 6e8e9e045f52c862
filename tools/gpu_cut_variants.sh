# A/B the PQ cut scan variants (tools/var/*.so): C3 step and scan kernel time, 3 rounds
mkdir -p gpurun_out
cp paper_1407_4764_b200/libotf_b200.so /tmp/otf_default.so
for round in 1 2 3; do
for v in tools/var/*.so; do
  cp $v paper_1407_4764_b200/libotf_b200.so
  timeout -k 10 300 python bench.py --config c3 --steps 50 --warmup 5 --no-cpu > gpurun_out/var.log 2>&1
  echo var=$(basename $v) $(tail -1 gpurun_out/var.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['ms_per_step']*1000,1), 'us/step scan', round(d['roofline']['kernel_ms']*1000,1), d['clocks']['sm_mhz'])" 2>&1 | tail -1)
done
done
cp /tmp/otf_default.so paper_1407_4764_b200/libotf_b200.so
