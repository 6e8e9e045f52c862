# per-CTA phase timeline of the PQ cut kernel (diagnostic build -DOTF_CUT_TRACE)
mkdir -p gpurun_out
OTF_NVCC_EXTRA="-DOTF_CUT_TRACE" python -c "from paper_1407_4764_b200 import _build; _build.build(force=True)"
timeout 600 python bench.py --config c3 --steps 1 --warmup 3 --no-cpu 2>&1 | grep -E "cutT|smpT" > gpurun_out/cut_trace_all.txt; grep cutT gpurun_out/cut_trace_all.txt > gpurun_out/cut_trace.txt; grep smpT gpurun_out/cut_trace_all.txt | tail -8
python - <<'PY'
import re
L = open("gpurun_out/cut_trace.txt").read().splitlines()[-148:]
keys = ["sample", "held", "threshold", "scan", "barrier", "select", "total"]
vals = {k: [] for k in keys}
for l in L:
    for k in keys:
        m = re.search(k + r" ([\d.]+)", l)
        vals[k].append(float(m.group(1)))
print(L[0][:60])
for k in keys:
    v = sorted(vals[k]); print(f"{k:8s} min {v[0]:.2f} med {v[len(v)//2]:.2f} max {v[-1]:.2f} us")
PY
python -c "from paper_1407_4764_b200 import _build; _build.build(force=True)"
