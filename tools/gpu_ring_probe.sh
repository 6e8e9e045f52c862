# PQ cut kernel ring diagnostics: per-CTA phase times (-DOTF_CUT_TRACE) with and without the
# scoring (-DOTF_CUT_NOCOMPUTE: the codes stream through the ring and are only read), C3 and C3x
mkdir -p gpurun_out
summ() {
python - "$1" <<'PY'
import re, sys
L = [l for l in open(sys.argv[1]).read().splitlines() if l.startswith("cutT")][-148:]
keys = ["sample", "held", "threshold", "scan", "barrier", "total"]
out = []
for k in keys:
    v = sorted(float(re.search(k + r" ([\d.]+)", l).group(1)) for l in L)
    out.append(f"{k} {v[len(v)//2]:.2f}")
print(sys.argv[1], " ".join(out))
PY
}
for extra in "$@"; do
  OTF_NVCC_EXTRA="-DOTF_CUT_TRACE $extra" python -c "from paper_1407_4764_b200 import _build; _build.build(force=True)" || exit 1
  for c in c3 c3x; do
    f=gpurun_out/ring_$(echo "$extra" | tr -c 'A-Za-z0-9' '_')_$c.txt
    timeout 600 python bench.py --config $c --steps 1 --warmup 3 --no-cpu --no-train 2>&1 | grep cutT > "$f"
    summ "$f"
  done
done
