"""Where does an M = 64 tcgen05 accumulator land in TMEM? (ts_probe_m64)"""
import os as _os, sys as _sys
_sys.path.insert(0, _os.path.dirname(_os.path.dirname(_os.path.abspath(__file__))))
import torch
from paper_2512_02371_b200 import _lib
L = _lib.load_diag()
g = torch.Generator().manual_seed(0)
n = 32
a = torch.randn(64, 16, generator=g).bfloat16().float().cuda()
b = torch.randn(16, n, generator=g).bfloat16().float().cuda()
ref = (a @ b).cpu()
for lb in (0, 64, 32):
    d = torch.zeros(128, n, device="cuda")
    st = L.ts_probe_m64(a.data_ptr(), b.data_ptr(), d.data_ptr(), n, lb, None)
    torch.cuda.synchronize()
    d = d.cpu()
    written = [(r, ) for r in range(128) if not torch.all(d[r] == -1.0)]
    rows = [r for r in range(128) if not torch.all(d[r] == -1.0)]
    print("lane_base", lb, "status", st, "written lanes", rows[:4], "...", rows[-4:] if rows else None, "count", len(rows))
    # match each written lane to a row of ref
    for r in rows[:3] + rows[-3:]:
        best = int(torch.argmin((ref - d[r]).abs().sum(1)))
        print("   lane", r, "-> ref row", best, "err", float((ref[best] - d[r]).abs().max()), "cols written", int((d[r] != -1).sum()))
