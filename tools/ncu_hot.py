"""Print the hottest SASS instructions (warp-stall samples) of a kernel in an
.ncu-rep:  python tools/ncu_hot.py REP KERNEL_REGEX [N]"""
import csv
import subprocess
import sys

rep, kern = sys.argv[1], sys.argv[2]
n = int(sys.argv[3]) if len(sys.argv) > 3 else 30
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "-k", f"regex:{kern}"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
hdr = rows[1]
si = hdr.index("Warp Stall Sampling (All Samples)")
ie = hdr.index("Instructions Executed")
body = []
for r in rows[2:]:
    if r and r[0] == "Kernel Name" and body:
        break
    if len(r) > si and r[si].replace(".", "").isdigit():
        body.append(r)
tot = sum(float(r[si] or 0) for r in body) or 1
print(f"total samples {tot:.0f}, instructions {len(body)}")
ranked = sorted(range(len(body)), key=lambda i: -float(body[i][si] or 0))[:n]
for i in sorted(ranked):
    r = body[i]
    print(f"{float(r[si] or 0) / tot * 100:5.1f}%  {i:5d} {r[ie]:>9} {r[1].strip()[:80]}")
