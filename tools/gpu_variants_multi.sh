# Multi-classifier GPU tests + full-size C5b timing for each tools/var/*.so variant.
cp paper_1407_4764_b200/libotf_b200.so /tmp/otf_default.so
for v in tools/var/*.so; do
  cp $v paper_1407_4764_b200/libotf_b200.so
  echo var=$(basename $v) test: $(timeout -k 10 300 python -m pytest tests/test_gpu_multi.py -x -q 2>&1 | grep -E "passed|failed|Error" | tail -2)
  for rep in 1 2; do
    timeout -k 10 600 python bench.py --config c5b --steps 5 --warmup 3 --no-cpu > gpurun_out/varm.log 2>&1
    tail -1 gpurun_out/varm.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('var=$(basename $v)', round(d['ms_per_step'],2), round(d['roofline']['kernel_ms'],2), round(d['roofline']['frac'],3), d['clocks'])" || tail -3 gpurun_out/varm.log
  done
done
cp /tmp/otf_default.so paper_1407_4764_b200/libotf_b200.so
