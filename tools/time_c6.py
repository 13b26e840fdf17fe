"""Large-factor resamples (config c6 geometries, 4K->540p): launch plan of
the fused kernel (rows per tile) or two-pass, and the time per 48 planes."""
import os as _os, sys as _sys
_sys.path.insert(0, _os.path.dirname(_os.path.dirname(_os.path.abspath(__file__))))
import ctypes, json, torch
from paper_2512_02371_b200 import _lib, axis, pipelines
L = _lib.load()
o = (ctypes.c_int * 8)()
for H, W, oh, ow in [(2048, 2048, 921, 921), (2048, 2048, 450, 450), (2048, 2048, 245, 245),
                     (2048, 2048, 143, 143), (2160, 3840, 540, 960)]:
    ra, ca = axis.lanczos3(H, oh, 0), axis.lanczos3(W, ow, 0)
    st = L.ts_separable_plan(ra.handle, ca.handle, 48, 1, o)
    x = torch.rand((48, H, W), device="cuda").bfloat16()
    for _ in range(3): y = pipelines.resample(x, oh, ow)
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(20): y = pipelines.resample(x, oh, ow)
    e.record(); torch.cuda.synchronize()
    ms = s.elapsed_time(e) / 20
    print(json.dumps({"cfg": f"{H}x{W}->{oh}x{ow}", "fused": st == 0,
                      "plan[nst,nmid,res,smem,R1,nb2,tiles,grid]": list(o) if st == 0 else None,
                      "ms": round(ms, 4), "GBps": round((x.numel() + y.numel()) * 2 / ms / 1e6)}), flush=True)
    del x, y
