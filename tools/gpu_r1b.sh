mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -m gpu > gpurun_out/pytest_gpu.log 2>&1; echo pytest=$?; tail -3 gpurun_out/pytest_gpu.log
python __graft_entry__.py > gpurun_out/smoke.log 2>&1; echo smoke=$?
for c in c2 c1 c3 c5a; do python bench.py --config $c > gpurun_out/bench_$c.log 2>&1; echo bench_$c=$?; done
