mkdir -p gpurun_out
for c in c2 c3; do
python bench.py --config $c --steps 5 --warmup 3 --no-cpu > gpurun_out/plain_$c.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_$c.csv python bench.py --config $c --steps 5 --warmup 3 --no-cpu > gpurun_out/ncu_$c.log 2>&1; echo ncu_$c=$?
done
ncu --set full --clock-control none --import-source on -k regex:"pq_scan|topk" -s 4 -c 2 -o gpurun_out/prof_c3 python bench.py --config c3 --steps 5 --warmup 3 --no-cpu > gpurun_out/ncu3.log 2>&1; echo ncu3=$?
