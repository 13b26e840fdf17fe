"""Per-source-line instruction counts (and stall samples) of an ncu report:
    python tools/ncu_lines.py REPORT.ncu-rep [N]"""
import csv
import subprocess
import sys
from collections import Counter

rep = sys.argv[1]
n = int(sys.argv[2]) if len(sys.argv) > 2 else 40
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
per, stall, text = Counter(), Counter(), {}
ie = sa = None
cur = None
fname = ""
for r in rows:
    if not r:
        continue
    if r[0] == "File Path":
        fname = r[1].split("/")[-1]
        continue
    if r[0] == "Function Name":
        continue
    if r[0] == "Line No":
        ie = r.index("Instructions Executed")
        sa = r.index("Warp Stall Sampling (All Samples)")
        continue
    if r[0]:
        try:
            cur = (fname, int(r[0]))
        except ValueError:
            continue
        text[cur] = r[1][:90]
        continue  # the cuda line row repeats its sass rows' totals
    if ie is not None and len(r) > ie and r[ie]:
        try:
            per[cur] += int(r[ie])
            stall[cur] += int(r[sa] or 0)
        except ValueError:
            pass
tot = sum(per.values())
stot = sum(stall.values()) or 1
print(f"total warp instructions {tot}, stall samples {stot}")
for l, v in per.most_common(n):
    print(f"{v:10d} {v / tot:5.3f} stall {stall[l] / stot:5.3f} {l[0][:12]:12s}{l[1]:5d} {text.get(l, '')}")
