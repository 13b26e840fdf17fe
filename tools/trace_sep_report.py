"""Median per-tile cycle offsets of the fused separable kernel's trace
(gpurun_out/trace.npy from tools/trace_sep.py), relative to the tile's
producer-start stamp, plus the steady-state period."""
import numpy as np
t = np.load("gpurun_out/trace.npy").astype(np.int64)  # [cta][tile][10]
names = ["prod: start", "prod: stage free -> TMA issued", "P1: input landed", "P1: issued",
         "E1: V acc seen", "E1: mid stored", "P2: mid seen", "P2: issued", "E2: H acc seen",
         "E2: store issued"]
rows = []
for c in range(t.shape[0]):
    for i in range(4, t.shape[1] - 1):
        if (t[c, i] == 0).any() or t[c, i + 1, 2] == 0:
            continue
        rows.append(np.concatenate([t[c, i] - t[c, i, 0], [t[c, i + 1, 2] - t[c, i, 2]]]))
r = np.array(rows)
for k, n in enumerate(names + ["period (P1 input landed)"]):
    print(f"{n:32s} {int(np.median(r[:, k])):7d}")
