mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_multi.py -q -x -p no:cacheprovider -k "rank_many" > gpurun_out/seg_tests.log 2>&1; echo seg_tests=$?; tail -15 gpurun_out/seg_tests.log
for v in "" "OTF_SEG_NO_CUT=1"; do
  env $v timeout 900 python bench.py --config c5b --steps 10 --warmup 3 --no-cpu > gpurun_out/seg_c5b.log 2>&1
  tail -1 gpurun_out/seg_c5b.log | python -c "import json,sys
d=json.loads(sys.stdin.read()); r=d['roofline']
print('c5b $v', round(d['ms_per_step'],3), 'ms/step kernel', round(r['kernel_ms'],3), 'ms frac', round(r['frac'],3), d['clocks']['sm_mhz'], d['clocks']['reasons'])"
done
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_seg.csv python bench.py --config c5b --steps 3 --warmup 3 --no-cpu > /dev/null 2>&1
python tools/launches.py gpurun_out/launches_seg.csv | grep otf
