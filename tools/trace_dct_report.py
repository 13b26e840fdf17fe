"""Median per-band cycle offsets of the DCT trace events (gpurun_out/trace_dct.npy,
written by tools/trace_dct.py), relative to the band's p=0 D1-seen stamp."""
import numpy as np
t = np.load("gpurun_out/trace_dct.npy").astype(np.int64)  # [cta][band][24]
names = {0: "D1 seen", 1: "C1 done", 2: "D2 q0 seen", 6: "D2 q1 seen", 3: "E2 done", 4: "D3 seen", 5: "E3 done"}
rows = []
for c in range(t.shape[0]):
    for b in range(2, t.shape[1] - 1):
        if t[c, b, 0] == 0 or t[c, b + 1, 0] == 0:
            continue
        base = t[c, b, 0]
        r = {"band period": t[c, b + 1, 0] - base}
        for p in range(2):
            for e, n in names.items():
                r[f"p{p} {n}"] = t[c, b, 12 * p + e] - base
        r["E4 start"] = t[c, b, 22] - base
        r["E4 stored"] = t[c, b, 23] - base
        rows.append(r)
keys = rows[0].keys()
for k in keys:
    v = np.array([r[k] for r in rows])
    print(f"{k:16s} {int(np.median(v)):8d}")
