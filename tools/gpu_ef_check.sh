cp paper_1407_4764_b200/libotf_b200.so /tmp/otf_default.so
for round in 1 2; do
for v in tools/var/*.so; do
  cp $v paper_1407_4764_b200/libotf_b200.so
  echo $(basename $v) $(timeout 300 python -m pytest tests/test_gpu_fullsize.py -q -k c2 2>&1 | tail -1)
done
done
cp /tmp/otf_default.so paper_1407_4764_b200/libotf_b200.so
