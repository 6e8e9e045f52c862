mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_pq_cut.py tests/test_gpu_fullsize.py -k "cut or c3" -q -x > gpurun_out/r2f_tests.log 2>&1; echo tests=$?; tail -1 gpurun_out/r2f_tests.log
timeout 600 python bench.py --config c3 --steps 50 --warmup 5 --no-cpu > gpurun_out/r2f_c3.log 2>&1; echo c3=$?
tail -1 gpurun_out/r2f_c3.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); r=d['roofline']; print('c3', round(d['ms_per_step']*1000,1), 'us/step scan', round(r['kernel_ms']*1000,1), 'us frac', round(r['frac'],3), 'e2e us', round(d['e2e']['ms_per_query']*1000,1))"
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r2f_launch_c3.csv python bench.py --config c3 --steps 5 --warmup 3 --no-cpu > /dev/null 2>&1
python tools/launches.py gpurun_out/r2f_launch_c3.csv | grep -E "otf::" | head -6
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"pq_lut_sample|pq_scan16_cut|topk_cut" -c 3 -o gpurun_out/r2f_c3scan -f python bench.py --config c3 --steps 1 --warmup 3 --no-cpu > gpurun_out/r2f_ncu.log 2>&1; echo ncu=$?
bash tools/gpu_cut_trace.sh
