mkdir -p gpurun_out
line() { tail -1 $1 | python -c "import json,sys
d=json.loads(sys.stdin.read()); r=d['roofline']
print('$2', 'step_ms', round(d['ms_per_step'],4), 'kernel_ms', round(r.get('kernel_ms',0),4), 'frac', round(r['frac'],3), 'e2e', round(d['e2e']['ms_per_query'],4), 'clk', d['clocks']['sm_mhz'])"; }

for v in "-DOTF_DC_R1=8" "-DOTF_DC_R1=16"; do
  OTF_NVCC_EXTRA="$v" python -c "from paper_1407_4764_b200 import _build; _build.build(force=True)" > /dev/null 2>&1
  for i in 1 2; do timeout 900 python bench.py --config c1 --steps 50 --warmup 5 --no-cpu > gpurun_out/c1r.log 2>&1; line gpurun_out/c1r.log "c1 $v"; done
done
