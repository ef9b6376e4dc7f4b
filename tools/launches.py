"""Summarise an ncu --metrics gpu__time_duration.sum --csv launch list:
python tools/launches.py file.csv [...]"""
import csv
import sys
from collections import defaultdict

for path in sys.argv[1:]:
    rows = list(csv.reader(open(path)))
    hdr, agg = None, defaultdict(list)
    for r in rows:
        if "Kernel Name" in r:
            hdr = r
            continue
        if hdr and len(r) == len(hdr):
            d = dict(zip(hdr, r))
            if d.get("Metric Name") == "gpu__time_duration.sum":
                agg[d["Kernel Name"][:64]].append(float(d["Metric Value"]))
    print(f"== {path}")
    tot = 0.0
    for k, v in sorted(agg.items(), key=lambda kv: -sum(kv[1])):
        if k.startswith("void at::"):
            continue
        tot += sum(v) / len(v)
        print(f"{len(v):4d} {sum(v) / len(v) / 1000:9.1f}us  {k}")
    print(f"     {tot / 1000:9.1f}us  (qd kernels, per-call average, summed)")
