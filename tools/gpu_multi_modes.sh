mkdir -p gpurun_out
for m in ${MODES:-0}; do
  OTF_MULTI_MODE=$m OTF_BENCH_ROWS=${ROWS:-4000000} timeout -k 10 300 python bench.py --config c5b --steps 5 --warmup 3 --no-cpu > gpurun_out/mm_$m.log 2>&1
  echo mode=$m $(grep -o '"kernel_ms": [0-9.]*' gpurun_out/mm_$m.log) $(grep -o '"clocks": {[^}]*}' gpurun_out/mm_$m.log)
done
