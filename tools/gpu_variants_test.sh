# Run the multi-classifier GPU tests against each tools/var/*.so variant, then time them.
cp paper_1407_4764_b200/libotf_b200.so /tmp/otf_default.so
for v in tools/var/*.so; do
  cp $v paper_1407_4764_b200/libotf_b200.so
  echo var=$(basename $v) test: $(timeout -k 10 300 python -m pytest tests/test_gpu_multi.py -x -q 2>&1 | tail -1)
done
cp /tmp/otf_default.so paper_1407_4764_b200/libotf_b200.so
bash tools/gpu_variants.sh
