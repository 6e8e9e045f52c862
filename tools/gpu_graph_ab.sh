# bench step with / without the CUDA-graph replay of the rank
mkdir -p gpurun_out
for c in c1 c2 c3 c5a; do
  for v in "OTF_X=1" "OTF_BENCH_NO_GRAPH=1"; do
    env $v timeout 600 python bench.py --config $c --steps 30 --warmup 5 --no-cpu > gpurun_out/g_$c.log 2>&1
    echo "$c $v $(tail -1 gpurun_out/g_$c.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['ms_per_step']*1000,1), 'us/step; launches', d['gpu_launches'], 'kernel', round(d['roofline']['kernel_ms']*1000,1), 'e2e', round(d['e2e']['ms_per_query']*1000,1))")"
  done
done
