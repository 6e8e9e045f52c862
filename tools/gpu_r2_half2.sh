mkdir -p gpurun_out
for v in "-DOTF_PQ_HALF_DIV=0" "-DOTF_PQ_HALF_DIV=8"; do
  echo "== $v"
  OTF_NVCC_EXTRA="$v -DOTF_CUT_TRACE" python -c "from paper_1407_4764_b200 import _build; _build.build(force=True)" > /dev/null 2>&1
  timeout 600 python bench.py --config c3 --steps 1 --warmup 3 --no-cpu 2>&1 | grep "cutT" | tail -148 > gpurun_out/ct.txt
  python - <<'PY'
import re
L = open("gpurun_out/ct.txt").read().splitlines()
keys = ["C", "sample", "held", "threshold", "scan", "barrier", "select", "total"]
for k in keys:
    v = sorted(float(re.search(k + r" ([\d.]+)", l).group(1)) for l in L)
    print(f"{k:9s} min {v[0]:.2f} med {v[len(v)//2]:.2f} max {v[-1]:.2f}")
PY
  OTF_NVCC_EXTRA="$v" python -c "from paper_1407_4764_b200 import _build; _build.build(force=True)" > /dev/null 2>&1
  timeout 600 python bench.py --config c3 --steps 50 --warmup 5 --no-cpu 2>&1 | tail -1 | cut -c100-140
done
