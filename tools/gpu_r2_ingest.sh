mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_ingest.py -q -x -p no:cacheprovider > gpurun_out/ing_tests.log 2>&1; echo ing_tests=$?; tail -15 gpurun_out/ing_tests.log
timeout 900 python tools/ingest_bench.py 100000000 /tmp > gpurun_out/ingest_bench.log 2>&1; echo ingest=$?; cat gpurun_out/ingest_bench.log | tail -6
OTF_INGEST_THREADS=8 timeout 900 python tools/ingest_bench.py 100000000 /tmp 2>&1 | tail -4
df -h /tmp | tail -1; nproc; free -g | head -2
