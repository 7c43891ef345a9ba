"""Summarise tools/sweep_decode.sh: one row per (context, budget)."""
import glob
import json
import os
import sys

rows = []
for f in sorted(glob.glob(os.path.join(sys.argv[1], "*.json"))):
    try:
        d = json.loads(open(f).read().strip().splitlines()[-1])
    except Exception:
        continue
    c = d["config"]
    rows.append((c["seq_len"], c["budget"], d["ms_per_step"], d["value"], d["roofline"]["frac"],
                 d["union_factor"], d["dense"]["ms_per_step"], d["dense"]["sparse_speedup"]))
print("| context | budget | sparse ms / step | GB/s | frac of peak | union / budget | dense ms / step | sparse / dense |")
print("|---|---|---|---|---|---|---|---|")
for r in sorted(rows):
    print(f"| {r[0] // 1024}K | {r[1]} | {r[2]:.3f} | {r[3]:.0f} | {r[4]:.3f} | {r[5]:.2f} | {r[6]:.3f} | {r[7]:.2f}x |")
