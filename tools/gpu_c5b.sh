mkdir -p gpurun_out
timeout -k 10 300 python -m pytest tests/test_gpu_multi.py -x -q -m gpu 2>&1 | tail -2
timeout -k 10 600 python bench.py --config c5b --steps 10 --warmup 3 > gpurun_out/bench_c5b.log 2>&1; echo bench=$?
tail -3 gpurun_out/bench_c5b.log | cut -c1-1500
