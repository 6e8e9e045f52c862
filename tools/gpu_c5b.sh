# C5b: multi-classifier tests (FP16 and TF32x3 forms), then the bench for both forms
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_multi.py -x -q > gpurun_out/c5b_tests.log 2>&1; echo tests_f16=$?; tail -3 gpurun_out/c5b_tests.log
OTF_MULTI_TF32=1 timeout 600 python -m pytest tests/test_gpu_multi.py -x -q > gpurun_out/c5b_tests_tf32.log 2>&1; echo tests_tf32=$?; tail -1 gpurun_out/c5b_tests_tf32.log
for v in "OTF_MULTI_X=0" "OTF_MULTI_TF32=1"; do
  env $v timeout 600 python bench.py --config c5b --steps 10 --warmup 3 --no-cpu > gpurun_out/c5b_v.log 2>&1
  echo "$v $(tail -1 gpurun_out/c5b_v.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); r=d['roofline']; print(round(d['ms_per_step'],2), 'ms/step kernel', round(r['kernel_ms'],2), 'frac', round(r['frac'],3), 'e2e', round(d['e2e']['ms_per_query'],2), d['clocks'])")"
done
