#!/bin/bash
# A/B of two prebuilt library variants (ab/libotf_<name>.so) on the bench configs given:
#   gpurun -- 'bash tools/gpu_ab.sh "new old new old" "c3 c3x"'
# each pass swaps the variant in as paper_1407_4764_b200/libotf_b200.so and prints ms_per_step.
mkdir -p gpurun_out
for v in $1; do
  cp "ab/libotf_$v.so" paper_1407_4764_b200/libotf_b200.so
  for c in $2; do
    ms=$(timeout 300 python bench.py --config "$c" --steps ${STEPS:-30} --warmup 5 --no-cpu --no-train 2>gpurun_out/ab_err.log |
      python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(d['ms_per_step'], d['roofline']['frac'])")
    echo "$v $c $ms"
  done
done
