# Time the c5b kernel for each tools/var/*.so variant (copied over the in-tree library in turn).
mkdir -p gpurun_out
cp paper_1407_4764_b200/libotf_b200.so /tmp/otf_default.so
for v in tools/var/*.so; do
  cp $v paper_1407_4764_b200/libotf_b200.so
  for m in ${MODES:-0}; do
    OTF_MULTI_MODE=$m OTF_BENCH_ROWS=${ROWS:-4000000} timeout -k 10 300 python bench.py --config c5b --steps 5 --warmup 3 --no-cpu > gpurun_out/var.log 2>&1
    echo var=$(basename $v) mode=$m $(grep -o '"kernel_ms": [0-9.]*' gpurun_out/var.log) $(grep -o '"clocks": {[^}]*}' gpurun_out/var.log) $(tail -c 300 gpurun_out/var.log | grep -i error)
  done
done
cp /tmp/otf_default.so paper_1407_4764_b200/libotf_b200.so
