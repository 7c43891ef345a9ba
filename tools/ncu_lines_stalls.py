"""Warp-stall samples of a kernel per CUDA source line, with the dominant
stall reasons: python tools/ncu_lines_stalls.py REP KERNEL_REGEX [N]"""
import csv
import subprocess
import sys

rep, kern = sys.argv[1], sys.argv[2]
n = int(sys.argv[3]) if len(sys.argv) > 3 else 40
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass", "-k", f"regex:{kern}"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
res, fname, hdr = [], None, None
for r in rows:
    if not r:
        continue
    if r[0] == "File Path":
        fname = r[1].split("/")[-1]
        continue
    if r[0] == "Line No":
        hdr = r
        continue
    if hdr is None or not r[0].isdigit():
        continue
    nm = len(hdr) - 4  # metric columns; the source text may contain unescaped quotes
    if len(r) < len(hdr):
        continue
    d = dict(zip(hdr[4:], r[-nm:]))
    s = float(d.get("Warp Stall Sampling (All Samples)", 0) or 0)
    if s <= 0:
        continue
    reasons = {k[6:]: float(v or 0) for k, v in d.items() if k.startswith("stall_") and "Not Issued" not in k}
    top = sorted(reasons.items(), key=lambda kv: -kv[1])[:3]
    res.append((s, fname, int(r[0]), r[1].strip()[:70], top))
tot = sum(x[0] for x in res) or 1
print(f"total samples {tot:.0f}")
for s, f, ln, src, top in sorted(res, key=lambda x: -x[0])[:n]:
    t = " ".join(f"{k}={v / s * 100:.0f}%" for k, v in top if v > 0)
    print(f"{s / tot * 100:5.1f}% {f}:{ln:<5d} {src:70s} {t}")
