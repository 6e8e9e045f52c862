for v in "OTF_DENSE_R1=8" "OTF_DENSE_R1=16" "OTF_DENSE_R1=32"; do
  env $v timeout 600 python bench.py --config c1 --steps 50 --warmup 5 --no-cpu > gpurun_out/d_c1.log 2>&1
  echo "$v $(tail -1 gpurun_out/d_c1.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['ms_per_step']*1000,1), 'us/step kernel', round(d['roofline']['kernel_ms']*1000,1), 'frac', round(d['roofline']['frac'],3))")"
done
