mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_dense_cut.py -q -x -p no:cacheprovider > gpurun_out/dc_tests.log 2>&1; echo dcut_tests=$?; tail -3 gpurun_out/dc_tests.log
timeout 600 python tools/latency_probe.py c1 c3 c2 > gpurun_out/lat.log 2>&1; echo lat=$?; cat gpurun_out/lat.log | tail -12
