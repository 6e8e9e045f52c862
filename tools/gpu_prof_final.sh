# refresh the profiles of configs whose kernels changed after r1c (c2: R=2 rows; c5b: FP16 groups of 8)
mkdir -p gpurun_out
for spec in "c2:dense_score|topk:2" "c5b:multi_score|topk:2"; do
  IFS=: read cfg kr cnt <<< "$spec"
  timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_r1c_$cfg.csv \
      python bench.py --config $cfg --steps 5 --warmup 3 --no-cpu > /dev/null 2>&1; echo launches_$cfg=$?
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:"$kr" -s 4 -c $cnt -o gpurun_out/prof_r1c_$cfg \
      python bench.py --config $cfg --steps 3 --warmup 3 --no-cpu > /dev/null 2>&1; echo full_$cfg=$?
done
