"""Copy a tools/profile_round.sh result set (gpurun_out/<R>/) into profiles/
(r02_* names) and regenerate the table of profiles/README.md.

    python tools/profiles_refresh.py gpurun_out/r02c
"""
import json
import os
import re
import shutil
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
src = sys.argv[1]
prof = os.path.join(ROOT, "profiles")
py = sys.executable
summ = os.path.join(ROOT, "tools", "ncu_summary.py")
caps = (("dct_c4", "-", "ncu_dct16_c4", 16, 3 * 2160 * 3840 * 4),
        ("sep_c2", "launches_c2.csv", "ncu_separable_c2", 16, None),
        ("f32_c1", "-", "ncu_f32_c1", 16, 3 * 1080 * 1920 * 4 + 3 * 540 * 960 * 4))
for rep, launches, out, frames, alg in caps:
    args = [py, summ, f"{rep}.ncu-rep", launches, out, str(frames)] + ([str(alg)] if alg else [])
    subprocess.run(args, cwd=src, check=True, capture_output=True)
    shutil.copy(os.path.join(src, f"{out}.json"), os.path.join(prof, f"r02_{out}.json"))
    with open(os.path.join(prof, f"r02_{out}_lines.txt"), "w") as f:
        subprocess.run([py, os.path.join(ROOT, "tools", "ncu_lines.py"),
                        os.path.join(src, f"{rep}.ncu-rep"), "12"], stdout=f, check=True)
for fn in os.listdir(src):
    if fn.startswith("bench_") and fn.endswith(".json"):
        shutil.copy(os.path.join(src, fn), os.path.join(prof, "r02_" + fn))
shutil.copy(os.path.join(src, "ncu_summary.json"), os.path.join(prof, "ncu_summary.json"))

names = {"c2": "c2 4K→1080p Lanczos-3", "c1": "c1 1080p f32 → 540p (K5, TMA, FMA pipe)",
         "c3-9": "c3 8K Gaussian 9", "c3-15": "c3 8K Gaussian 15", "c3-21": "c3 8K Gaussian 21",
         "c3-31": "c3 8K Gaussian 31", "c4": "c4 4K DCT-16 denoise (hard)",
         "c5": "c5 512 frames resample+filter", "c6-143": "c6 2048² → 143²",
         "c6-245": "c6 2048² → 245²", "c6-450": "c6 2048² → 450²", "c6-921": "c6 2048² → 921²"}
tab = []
for c, n in names.items():
    d = json.load(open(os.path.join(prof, f"r02_bench_{c}.json")))
    r, cl, su = d["roofline"], d["clocks"], d["sustained"]
    tab.append(f"| {n} | {d['value']:,.0f} | {r['frac']:.3f} | {r['avg_launch_ms'] * 1e3:.0f} µs | "
               f"{(r['traffic'] or 0) / r['alg_bytes_per_launch']:.2f} | {su['roofline_frac']:.3f} "
               f"({su['sm_mhz']:.0f} MHz {', '.join(su['reasons'])}) | {d['e2e']['value']:,.0f} | "
               f"{cl['sm_mhz']:.0f} {', '.join(cl['reasons'])} |")
ref = json.load(open(os.path.join(prof, "r02_bench_reference_c2.json")))
readme = os.path.join(prof, "README.md")
s = open(readme).read()
a = s.index("| config | value (Mpixel/s) | frac (timed)")
b = s.index("* CPU baseline (`cpu_baseline`")
hdr = ("| config | value (Mpixel/s) | frac (timed) | kernel avg | traffic/alg | sustained frac | "
       "e2e (Mpixel/s) | SM MHz (timed), reasons |\n|---|---|---|---|---|---|---|---|\n")
s = (s[:a] + hdr + "\n".join(tab) +
     f"\n| reference arm (tensorsel interp, 16 cores, c2) | {ref['value']} | — | — | — | — | — | — |\n\n"
     + s[b:])
cp = {c: json.load(open(os.path.join(prof, f"r02_bench_{c}.json")))["cpu_baseline"]["value"]
      for c in ("c2", "c1", "c4", "c5")}
s = re.sub(r"(\* CPU baseline \(`cpu_baseline`, the numpy oracle over all 16 host cores\):\n  )"
           r"c2 [0-9.]+, c1 [0-9.]+, c4 [0-9.]+, c5 [0-9.]+",
           rf"\1c2 {cp['c2']}, c1 {cp['c1']}, c4 {cp['c4']}, c5 {cp['c5']}", s)
open(readme, "w").write(s)
for k in ("ncu_separable_c2", "ncu_f32_c1", "ncu_dct16_c4"):
    d = json.load(open(os.path.join(prof, f"r02_{k}.json")))
    print(k, round(d["duration_us"], 1), "us", round(d["traffic_over_alg"], 3), "x alg")
