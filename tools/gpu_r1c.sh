mkdir -p gpurun_out
python bench.py --config c1 --steps 5 --warmup 3 --no-cpu > gpurun_out/plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_c1.csv python bench.py --config c1 --steps 5 --warmup 3 --no-cpu > gpurun_out/ncu1.log 2>&1; echo ncu1=$?
ncu --set full --clock-control none --import-source on -k regex:"dense_score|topk" -s 4 -c 2 -o gpurun_out/prof_c1 python bench.py --config c1 --steps 5 --warmup 3 --no-cpu > gpurun_out/ncu2.log 2>&1; echo ncu2=$?
