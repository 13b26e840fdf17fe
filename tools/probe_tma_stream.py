import os as _os, sys as _sys
_sys.path.insert(0, _os.path.dirname(_os.path.dirname(_os.path.abspath(__file__))))
import json, torch
from paper_2512_02371_b200 import _lib
L = _lib.load_diag()
x = torch.rand((48, 2160, 3840), device="cuda").bfloat16()
def run(rows, nbox, nr, grid=148, n=10):
    f = lambda: _lib.check(L.ts_probe_tma(x.data_ptr(), 48, 2160, 3840, rows, nbox, nr, grid, None))
    for _ in range(2): f()
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(n): f()
    e.record(); torch.cuda.synchronize()
    ms = s.elapsed_time(e) / n
    print(json.dumps({"rows": rows, "nbox": nbox, "nr": nr, "grid": grid, "kb_inflight": nr * rows * 128 * nbox // 1024,
                      "GBps": round(x.numel() * 2 / ms / 1e6, 1)}), flush=True)
for rows, nbox, nr in [(16, 4, 19), (16, 4, 24), (16, 4, 8), (32, 4, 10), (64, 4, 5), (16, 2, 32), (32, 2, 20),
                       (128, 2, 6), (136, 2, 6), (64, 2, 12), (16, 1, 32), (256, 1, 6), (64, 4, 6), (32, 4, 6), (16, 4, 12)]:
    run(rows, nbox, nr)
run(16, 4, 19, grid=296)
