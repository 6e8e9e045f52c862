mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_binary_cluster.py -q -x -p no:cacheprovider > gpurun_out/bc_tests.log 2>&1; echo bc_tests=$?; tail -15 gpurun_out/bc_tests.log
timeout 900 python -m pytest tests -m gpu -q -x -p no:cacheprovider -k "binary or bin" > gpurun_out/bc_tests2.log 2>&1; echo bin_tests=$?; tail -3 gpurun_out/bc_tests2.log
for v in "" "OTF_BIN_NO_CLUSTER=1"; do
  env $v timeout 900 python bench.py --config c5a --steps 20 --warmup 3 --no-cpu > gpurun_out/bc_c5a.log 2>&1
  tail -1 gpurun_out/bc_c5a.log | python -c "import json,sys
d=json.loads(sys.stdin.read()); r=d['roofline']
print('c5a $v', round(d['ms_per_step'],3), 'ms/step kernel', round(r['kernel_ms'],3), 'ms frac', round(r['frac'],3), 'e2e ms', round(d['e2e']['ms_per_query'],3), d['clocks']['sm_mhz'], d['clocks']['reasons'])"
done
