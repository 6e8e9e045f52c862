"""Top stall-sampled SASS lines of one kernel in an .ncu-rep (ncu --page source --csv)."""
import csv
import subprocess
import sys

rep, kern = sys.argv[1], sys.argv[2]
n = int(sys.argv[3]) if len(sys.argv) > 3 else 25
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "-k", f"regex:{kern}", "--print-source", "sass,cuda"],
                     capture_output=True, text=True).stdout.splitlines()
rows = list(csv.reader(out))
hdr_i = next(i for i, r in enumerate(rows) if "Address" in r or "Source" in r)
h = rows[hdr_i]
isrc = h.index("Source")
iss = h.index("Warp Stall Sampling (All Samples)")
data = []
for r in rows[hdr_i + 1:]:
    if len(r) != len(h):
        continue
    try:
        s = int(r[iss] or 0)
    except ValueError:
        continue
    data.append((s, r[isrc][:110]))
tot = sum(d[0] for d in data)
print("total samples", tot)
for s, src in sorted(data, reverse=True)[:n]:
    print(f"{s:6d} {100*s/max(tot,1):5.1f}%  {src}")
