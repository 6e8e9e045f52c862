mkdir -p gpurun_out
line() { tail -1 $1 | python -c "import json,sys
d=json.loads(sys.stdin.read()); r=d['roofline']
print('$2', 'step_ms', round(d['ms_per_step'],4), 'kernel_ms', round(r.get('kernel_ms',0),4), 'frac', round(r['frac'],3), 'clk', d['clocks']['sm_mhz'])"; }
for v in "-DOTF_DC_HOLD_SMALL=1" "-DOTF_DC_HOLD_SMALL=4" "-DOTF_DC_HOLD_SMALL=1" "-DOTF_DC_HOLD_SMALL=4"; do
  OTF_NVCC_EXTRA="$v" python -c "from paper_1407_4764_b200 import _build; _build.build(force=True)" > /dev/null 2>&1
  for c in c2 c4; do timeout 900 python bench.py --config $c --steps 20 --warmup 5 --no-cpu --no-train > gpurun_out/hold.log 2>&1; line gpurun_out/hold.log "$c $v"; done
done
python -c "from paper_1407_4764_b200 import _build; _build.build(force=True)" > /dev/null 2>&1
