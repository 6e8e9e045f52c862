mkdir -p gpurun_out
c3line() { tail -1 $1 | python -c "import json,sys
d=json.loads(sys.stdin.read()); r=d['roofline']
print('$2', round(d['ms_per_step']*1000,1), 'us/step kernel', round(r['kernel_ms']*1000,1), 'us frac', round(r['frac'],3), 'e2e us', round(d['e2e']['ms_per_query']*1000,1), d['clocks']['sm_mhz'], d['clocks']['reasons'])"; }
timeout 600 python bench.py --config c3 --steps 50 --warmup 5 --no-cpu > gpurun_out/pq_c3.log 2>&1; c3line gpurun_out/pq_c3.log "c3 b1s4"
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_pq.csv python bench.py --config c3 --steps 5 --warmup 3 --no-cpu > /dev/null 2>&1
python tools/launches.py gpurun_out/launches_pq.csv | grep otf
for v in "-DOTF_CUT_BATCHES=2 -DOTF_CUT_STAGES=2" "-DOTF_CUT_BATCHES=1 -DOTF_CUT_STAGES=3" "-DOTF_CUT_BATCHES=2 -DOTF_CUT_STAGES=3"; do
  OTF_NVCC_EXTRA="$v" python -c "from paper_1407_4764_b200 import _build; _build.build(force=True)" > /dev/null 2>&1
  timeout 600 python bench.py --config c3 --steps 50 --warmup 5 --no-cpu > gpurun_out/pq_c3v.log 2>&1; c3line gpurun_out/pq_c3v.log "c3 $v"
done
timeout 600 python -m pytest tests/test_gpu_pq_cut.py -q -x -p no:cacheprovider 2>&1 | tail -2
python -c "from paper_1407_4764_b200 import _build; _build.build(force=True)" > /dev/null 2>&1
