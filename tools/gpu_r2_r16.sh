mkdir -p gpurun_out
line() { tail -1 $1 | python -c "import json,sys
d=json.loads(sys.stdin.read()); r=d['roofline']
print('$2', 'step_ms', round(d['ms_per_step'],4), 'kernel_ms', round(r.get('kernel_ms',0),4), 'frac', round(r['frac'],3), 'clk', d['clocks']['sm_mhz'])"; }
for v in "-DOTF_DC_R16=1" "-DOTF_DC_R16=2" "-DOTF_DC_R16=4"; do
  OTF_NVCC_EXTRA="$v" python -c "from paper_1407_4764_b200 import _build; _build.build(force=True)" > gpurun_out/build_$v.log 2>&1 || tail -3 gpurun_out/build_$v.log
  for c in c2 c4; do timeout 900 python bench.py --config $c --steps 20 --warmup 5 --no-cpu --no-train > gpurun_out/r16.log 2>&1; line gpurun_out/r16.log "$c $v"; done
done
python -c "from paper_1407_4764_b200 import _build; _build.build(force=True)" > /dev/null 2>&1
