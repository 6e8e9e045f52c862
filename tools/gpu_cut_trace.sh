# per-CTA phase timeline of the fused PQ cut kernel (diagnostic build -DOTF_CUT_TRACE)
mkdir -p gpurun_out
OTF_NVCC_EXTRA="-DOTF_CUT_TRACE" python -c "from paper_1407_4764_b200 import _build; _build.build(force=True)"
timeout 600 python bench.py --config c3 --steps 1 --warmup 3 --no-cpu 2>&1 | grep "cutT" > gpurun_out/cut_trace.txt
python - <<'PY'
import re, statistics as st
L = open("gpurun_out/cut_trace.txt").read().splitlines()[-64:]
keys = ["sample", "threshold", "scan", "barrier", "select", "rank", "total"]
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
