# Round-2 profiles: per config the ncu launch list and one --set full capture of the rank
# path's kernels; the cut kernel's phase trace; compute-sanitizer over every kernel family.
mkdir -p gpurun_out
for spec in "c4:dense_score|topk:2" "c3:pq_rank_cut|pq_build_lut:2" "c1:dense_score|topk:2" "c5a:bin_score|topk:3" "c5b:multi_score|topk_seg|topk:2"; do
  IFS=: read cfg kr cnt <<< "$spec"
  timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_r2_$cfg.csv \
      python bench.py --config $cfg --steps 5 --warmup 3 --no-cpu --no-train > /dev/null 2>&1; echo launches_$cfg=$?
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:"$kr" -s 4 -c $cnt -o gpurun_out/prof_r2_$cfg \
      python bench.py --config $cfg --steps 3 --warmup 3 --no-cpu --no-train > /dev/null 2>&1; echo full_$cfg=$?
done
bash tools/gpu_cut_trace.sh
bash tools/gpu_sanitize.sh
