import os as _os, sys as _sys
_sys.path.insert(0, _os.path.dirname(_os.path.dirname(_os.path.abspath(__file__))))
import torch, json
from paper_2512_02371_b200 import _lib
L = _lib.load_diag()
c = torch.zeros(1, dtype=torch.int64, device="cuda")
cases = []
for am, bm in ((0, 0), (1, 0), (0, 1), (1, 1), (2, 0), (2, 1)):
    for n in (16, 64, 112, 128, 240, 256):
        for nacc in (1, 2):
            if n * nacc <= (384 if am == 2 else 512): cases.append((am, bm, n, nacc))
for am, bm, n, nacc in cases:
    for rep in range(2):
        _lib.check(L.ts_probe_issue2(am, bm, n, 128, nacc, c.data_ptr(), None)); torch.cuda.synchronize()
    cyc = c.item() / 128
    print(json.dumps({"a": am, "b": bm, "n": n, "nacc": nacc, "cyc_per_mma": round(cyc, 1),
                      "pct_peak": round(100 * 128 * n * 16 / cyc / 8192, 1)}), flush=True)
