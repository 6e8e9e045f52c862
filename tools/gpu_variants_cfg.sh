# Time one bench config for each tools/var/*.so variant: CFG=c3 bash tools/gpu_variants_cfg.sh
mkdir -p gpurun_out
cp paper_1407_4764_b200/libotf_b200.so /tmp/otf_default.so
for v in tools/var/*.so; do
  cp $v paper_1407_4764_b200/libotf_b200.so
  for rep in 1 2; do
    timeout -k 10 300 python bench.py --config ${CFG:-c3} --steps ${STEPS:-20} --warmup 3 --no-cpu > gpurun_out/varc.log 2>&1
    tail -1 gpurun_out/varc.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('var=$(basename $v)', round(d['ms_per_step'],4), round(d['roofline']['kernel_ms'],4), round(d['roofline']['frac'],3), d['clocks']['sm_mhz'])" || tail -3 gpurun_out/varc.log
  done
done
cp /tmp/otf_default.so paper_1407_4764_b200/libotf_b200.so
