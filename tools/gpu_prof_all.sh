# Refresh profiles/: per config a plain run, the ncu launch list and one --set full capture.
mkdir -p gpurun_out
for spec in "c1:dense_score|topk" "c2:dense_score|topk" "c3:pq_scan|topk" "c3e:pq_encode_kernel" "c5a:bin_score"; do
  cfg=${spec%%:*}; kr=${spec#*:}
  CFG=$cfg KREGEX="$kr" TAG=r1 timeout 900 bash tools/gpu_prof_one.sh
done
