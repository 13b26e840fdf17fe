"""Per-group timeline of the DCT-16 strip kernel (diagnostics build:
clock64 stamps, ts_debug_trace): median cycles of each stage of the chain.

    make -C paper_2512_02371_b200/csrc diag
    python tools/dct_trace.py [frames]

Events per group i (epilogue / MMA warp): 0 D1 seen (C1 start), 1 C1 done,
2/3 D2 phase 0/1 seen, 4 E2 done, 5 D3 seen, 6 E3 done, 7 D4 seen (E4
start), 8 D4 read; 9 S3 issue, 10 S5 issue, 11 E3 seen, 12 S7 issue."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
os.environ.setdefault("TSB_LIB_PATH", os.path.join(ROOT, "paper_2512_02371_b200", "_native",
                                                   "libtsb200_diag.so"))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2512_02371_b200 import _lib, pipelines  # noqa: E402

F = int(sys.argv[1]) if len(sys.argv) > 1 else 16
C, G = 8, 48
x = torch.rand((3 * F, 2160, 3840), device="cuda").bfloat16()
pipelines.denoise_dct16(x, 0.15)
buf = torch.zeros((C, G, 16), dtype=torch.int64, device="cuda")
lib = _lib.load_diag()
_lib.check(lib.ts_debug_trace(buf.data_ptr(), C, G))
pipelines.denoise_dct16(x, 0.15)
torch.cuda.synchronize()
_lib.check(lib.ts_debug_trace(None, 0, 0))
t = buf.cpu().numpy()
np.save(os.path.join(ROOT, "gpurun_out", "dct_trace.npy"), t)
names = {1: "C1 done", 2: "D2 q0 seen", 3: "D2 q1 seen", 4: "E2 done", 5: "D3 seen",
         6: "E3 done", 7: "D4 seen (E4)", 8: "D4 read", 9: "S3 issue", 10: "S5 issue",
         11: "E3 seen (MMA)", 12: "S7 issue"}
rows = []
for c in range(C):
    for g in range(2, G - 1):
        if t[c, g, 0] == 0 or t[c, g + 1, 0] == 0:
            continue
        base = t[c, g, 0]
        r = {"group period": t[c, g + 1, 0] - base}
        r.update({n: t[c, g, e] - base for e, n in names.items()})
        rows.append(r)
print(f"{len(rows)} groups; cycles after 'D1 seen' (median):")
for k in rows[0]:
    print(f"  {k:16s} {int(np.median([r[k] for r in rows])):8d}")
