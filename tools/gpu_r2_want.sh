mkdir -p gpurun_out
line() { tail -1 $1 | python -c "import json,sys
d=json.loads(sys.stdin.read()); r=d['roofline']
print('$2', 'step_ms', round(d['ms_per_step'],4), 'kernel_ms', round(r.get('kernel_ms',0),4), 'frac', round(r['frac'],3), 'clk', d['clocks']['sm_mhz'])"; }
for v in "-DOTF_CUT_WANT16=32" "-DOTF_CUT_WANT16=25" "-DOTF_CUT_WANT16=20"; do
  OTF_NVCC_EXTRA="$v" python -c "from paper_1407_4764_b200 import _build; _build.build(force=True)" > /dev/null 2>&1
  for c in c1 c3 c2; do timeout 900 python bench.py --config $c --steps 50 --warmup 5 --no-cpu > gpurun_out/want.log 2>&1; line gpurun_out/want.log "$c $v"; done
done
python -c "from paper_1407_4764_b200 import _build; _build.build(force=True)" > /dev/null 2>&1
timeout 1500 python tools/stress_cut.py 24 2>&1 | tail -3
