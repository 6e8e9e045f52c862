# A/B: PQ cut path (default) vs the bins path (OTF_PQ_NO_CUT=1) on C3, interleaved
for round in 1 2 3; do
  for mode in cut bins; do
    if [ $mode = bins ]; then export OTF_PQ_NO_CUT=1; else unset OTF_PQ_NO_CUT; fi
    timeout 300 python bench.py --config c3 --steps 100 --warmup 10 --no-cpu > gpurun_out/ab.log 2>&1
    echo $mode $(tail -1 gpurun_out/ab.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['ms_per_step']*1000,1), 'us/step kernel', round(d['roofline']['kernel_ms']*1000,1), 'e2e', round(d['e2e']['ms_per_query']*1000,1))")
  done
done
unset OTF_PQ_NO_CUT
