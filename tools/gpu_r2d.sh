# PQ cut path: parity tests, C3 bench, launch list
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_pq_cut.py tests/test_gpu_fullsize.py -q -x -k "cut or c3" > gpurun_out/r2d_tests.log 2>&1; echo tests=$?; tail -3 gpurun_out/r2d_tests.log
timeout 600 python bench.py --config c3 --steps 50 --warmup 5 --no-cpu > gpurun_out/r2d_c3.log 2>&1; echo c3=$?
tail -1 gpurun_out/r2d_c3.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); r=d['roofline']; print('c3', round(d['ms_per_step']*1000,1), 'us/step scan', round(r['kernel_ms']*1000,1), 'us frac', round(r['frac'],3), 'e2e us', round(d['e2e']['ms_per_query']*1000,1), d['clocks'])"
OTF_PQ_NO_CUT=1 timeout 600 python bench.py --config c3 --steps 50 --warmup 5 --no-cpu > gpurun_out/r2d_c3_nocut.log 2>&1
tail -1 gpurun_out/r2d_c3_nocut.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); r=d['roofline']; print('c3 nocut', round(d['ms_per_step']*1000,1), 'us/step scan', round(r['kernel_ms']*1000,1))"
OTF_BENCH_STEPS_NOTE=1 timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r2d_launch_c3.csv python bench.py --config c3 --steps 5 --warmup 3 --no-cpu > /dev/null 2>&1
python tools/launches.py gpurun_out/r2d_launch_c3.csv | grep -E "otf::" | head -6
