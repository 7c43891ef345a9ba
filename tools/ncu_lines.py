"""Per-CUDA-source-line totals of an .ncu-rep kernel (needs -lineinfo):
    python tools/ncu_lines.py REP KERNEL_REGEX [N] [--by instr|samples]"""
import csv
import subprocess
import sys

rep, kern = sys.argv[1], sys.argv[2]
n = int(sys.argv[3]) if len(sys.argv) > 3 and sys.argv[3].isdigit() else 30
by = "samples" if "samples" in sys.argv else "instr"
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source=cuda,sass",
                      "-k", f"regex:{kern}"], capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
fname = ""
hdr = None
lines = []
seen_kernel = 0
for r in rows:
    if not r:
        continue
    if r[0] == "File Path":
        fname = r[1].split("/")[-1]
        continue
    if r[0] == "Function Name":
        seen_kernel += 1
        continue
    if r[0] == "Line No":
        hdr = r
        continue
    if hdr and r[0] and r[0].isdigit():
        si = hdr.index("Warp Stall Sampling (All Samples)")
        ie = hdr.index("Instructions Executed")
        fl = lambda x: float(x) if x.replace(".", "", 1).isdigit() else 0.0
        lines.append((fname, int(r[0]), r[1].strip()[:70], fl(r[si]), fl(r[ie])))
tot_s = sum(x[3] for x in lines) or 1
tot_i = sum(x[4] for x in lines) or 1
key = (lambda x: -x[3]) if by == "samples" else (lambda x: -x[4])
print(f"samples {tot_s:.0f}, warp-instructions {tot_i:.0f}")
for f, ln, src, s, i in sorted(lines, key=key)[:n]:
    print(f"{s / tot_s * 100:5.1f}% smp {i / tot_i * 100:5.1f}% ins  {f}:{ln:<5d} {src}")
