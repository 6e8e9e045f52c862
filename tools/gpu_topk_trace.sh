# per-phase timing of the top-k kernel (diagnostic build with -DOTF_TOPK_TRACE)
mkdir -p gpurun_out
OTF_NVCC_EXTRA="-DOTF_TOPK_TRACE" python -c "from paper_1407_4764_b200 import _build; _build.build(force=True)"
for c in c1 c3 c5a; do
  timeout 600 python bench.py --config $c --steps 1 --warmup 3 --no-cpu 2>&1 | grep "topk cta" > gpurun_out/trace_$c.txt
  python - $c <<'PY'
import sys, re
c = sys.argv[1]
L = [l for l in open(f"gpurun_out/trace_{c}.txt")]
L = L[-148:]
rec = []
for l in L:
    m = re.search(r"cta (\d+) C=(\d+): start (\d+) gend (\d+) hits (\d+) maxwarp (\d+) B ([\d.]+) gather ([\d.]+)", l)
    rec.append(tuple(int(m.group(i)) for i in (1, 3, 4)) + (float(m.group(7)), float(m.group(8)), int(m.group(5)), int(m.group(6))))
t0 = min(r[1] for r in rec)
rec.sort(key=lambda r: -r[2])
print(c, "start skew us", (max(r[1] for r in rec) - t0) / 1e3, "slowest gather ends (cta, end us, B, gather):",
      [(r[0], round((r[2] - t0) / 1e3, 2), r[3], r[4], r[5], r[6]) for r in rec[:5]], "hits median", sorted(r[5] for r in rec)[74], "median end", round((rec[len(rec)//2][2]-t0)/1e3, 2))
PY
done
