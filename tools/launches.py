"""Summarise an ncu --metrics gpu__time_duration.sum --csv launch list: per-kernel count/mean/min."""
import csv
import sys
from collections import defaultdict

agg = defaultdict(list)
hdr = None
for r in csv.reader(open(sys.argv[1])):
    if "Kernel Name" in r:
        hdr = r
        continue
    if hdr and len(r) == len(hdr):
        d = dict(zip(hdr, r))
        if d.get("Metric Name") == "gpu__time_duration.sum":
            agg[d["Kernel Name"][:80]].append(float(d["Metric Value"].replace(",", "")))
for k, v in agg.items():
    print(f"{len(v):4d} mean {sum(v)/len(v)/1000:10.2f} us  min {min(v)/1000:9.2f} us  {k}")
