import os as _os, sys as _sys
_sys.path.insert(0, _os.path.dirname(_os.path.dirname(_os.path.abspath(__file__))))
import json, torch
from paper_2512_02371_b200 import _lib
L = _lib.load_diag()
c = torch.zeros(1, dtype=torch.int64, device="cuda")
for x in (16, 32):
    for warps in (4, 8, 16):
        cols, reps = 256, 32
        for _ in range(2):
            _lib.check(L.ts_probe_tmem_ld(x, warps, cols, reps, c.data_ptr(), None)); torch.cuda.synchronize()
        cyc = c.item()
        byts = 128 * cols * 4 * reps
        print(json.dumps({"x": x, "warps": warps, "cycles": cyc, "B_per_cycle": round(byts / cyc, 1)}), flush=True)
