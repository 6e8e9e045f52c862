# per-CTA phase timeline of the fused dense cut kernel (diagnostic build -DOTF_DCUT_TRACE)
mkdir -p gpurun_out
OTF_NVCC_EXTRA="-DOTF_DCUT_TRACE" python -c "from paper_1407_4764_b200 import _build; _build.build(force=True)"
timeout 600 python bench.py --config ${CFG:-c1} --steps 1 --warmup 3 --no-cpu 2>&1 | grep "dcutT" > gpurun_out/dcut_trace.txt
python - <<'PY'
import re
L = open("gpurun_out/dcut_trace.txt").read().splitlines()[-296:]
keys = ["sample", "barrier1", "scan", "barrier2", "select", "rank", "total"]
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
