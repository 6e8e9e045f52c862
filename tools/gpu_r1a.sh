mkdir -p gpurun_out
set -x
nvidia-smi --query-gpu=clocks.sm,clocks.max.sm --format=csv
python __graft_entry__.py > gpurun_out/smoke.log 2>&1; echo smoke=$?
python bench.py > gpurun_out/bench_c2.log 2>&1; echo bench=$?
python bench.py --config c1 --no-cpu > gpurun_out/bench_c1.log 2>&1; echo bench1=$?
python bench.py --config c3 --no-cpu > gpurun_out/bench_c3.log 2>&1; echo bench3=$?
python bench.py --steps 5 --warmup 3 --no-cpu > gpurun_out/plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_c2.csv python bench.py --steps 5 --warmup 3 --no-cpu > gpurun_out/ncu1.log 2>&1; echo ncu1=$?
ncu --set full --clock-control none --import-source on -k regex:"dense_score|topk" -s 6 -c 2 -o gpurun_out/prof_c2 python bench.py --steps 5 --warmup 3 --no-cpu > gpurun_out/ncu2.log 2>&1; echo ncu2=$?
