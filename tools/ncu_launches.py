"""Summarise an ncu --metrics gpu__time_duration.sum launch list (csv):
    python tools/ncu_launches.py launches.csv"""
import csv
import sys
from collections import OrderedDict

rows = list(csv.reader(open(sys.argv[1])))
hdr = None
agg = OrderedDict()
for r in rows:
    if "Kernel Name" in r:
        hdr = r
        continue
    if hdr and len(r) == len(hdr):
        d = dict(zip(hdr, r))
        if d.get("Metric Name") == "gpu__time_duration.sum":
            v = float(d["Metric Value"]) * (1e-3 if d["Metric Unit"] == "ns" else 1.0)
            agg.setdefault(d["Kernel Name"].split("(")[0][:50], []).append(v)
tot = sum(sum(v) for k, v in agg.items() if "dsk::" in k or "k_" in k)
print(f"{'kernel':50s} {'n':>5s} {'mean us':>9s} {'share of dsk':>12s}")
for k, v in agg.items():
    mine = "dsk::" in k or "k_" in k
    print(f"{k:50s} {len(v):5d} {sum(v)/len(v):9.2f} {(sum(v)/tot*100 if mine else 0):11.1f}%")
