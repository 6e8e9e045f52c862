# PQ rank path: parity tests, then c3 with the float32-screening scan variants and the float64 scan
mkdir -p gpurun_out
timeout 600 python -m pytest tests -m gpu -x -q -k "pq or PQ or c3" > gpurun_out/pq_tests.log 2>&1; echo tests=$?
tail -1 gpurun_out/pq_tests.log
for v in ${PQ_VARIANTS:-"OTF_PQ_ROWS=4" "OTF_PQ_ROWS=2"}; do
env $v timeout 600 python bench.py --config c3 --steps 50 --warmup 5 --no-cpu > gpurun_out/pq_v.log 2>&1
env $v ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_pqv.csv python bench.py --config c3 --steps 5 --warmup 3 --no-cpu > /dev/null 2>&1
echo "$v $(tail -1 gpurun_out/pq_v.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['ms_per_step']*1000,1), 'us/step e2e', round(d['e2e']['ms_per_query']*1000,1))")"
python tools/launches.py gpurun_out/launches_pqv.csv | grep -E "pq_scan16_f32|topk"
done
