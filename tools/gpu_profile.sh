# Round profiling session on one B200 (run via gpurun). Plain runs first, ncu only after the
# identical command exited 0 (B200_PROFILING.md). Outputs land in gpurun_out/.
mkdir -p gpurun_out
TAG=${TAG:-r1}
for c in c2 c1 c3 c5a; do
  python bench.py --config $c > gpurun_out/bench_${TAG}_$c.log 2>&1; echo bench_$c=$?
done
python bench.py --impl reference > gpurun_out/bench_${TAG}_reference_c2.log 2>&1; echo ref=$?
for c in c2 c1 c3 c5a; do
  python bench.py --config $c --steps 5 --warmup 3 --no-cpu > gpurun_out/plain_$c.log 2>&1 && \
  ncu --metrics gpu__time_duration.sum --clock-control none --csv \
      --log-file gpurun_out/launches_${TAG}_$c.csv \
      python bench.py --config $c --steps 5 --warmup 3 --no-cpu > gpurun_out/ncu_l_$c.log 2>&1
  echo launches_$c=$?
  ncu --set full --clock-control none --import-source on \
      -k regex:"dense_score|pq_scan|bin_score|topk" -s 4 -c 2 -o gpurun_out/prof_${TAG}_$c \
      python bench.py --config $c --steps 5 --warmup 3 --no-cpu > gpurun_out/ncu_f_$c.log 2>&1
  echo full_$c=$?
done
