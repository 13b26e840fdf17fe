"""Per-pass timing of the two-pass resample (config c6 geometries and
4K->540p): vertical and horizontal ts_axis_pass launches timed separately
with CUDA events, 48 planes, bf16 in/out."""
import os as _os, sys as _sys
_sys.path.insert(0, _os.path.dirname(_os.path.dirname(_os.path.abspath(__file__))))
import json, torch
from paper_2512_02371_b200 import _lib, axis as _axis, pipelines


def t(fn, n=20):
    for _ in range(3): fn()
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(n): fn()
    e.record(); torch.cuda.synchronize()
    return s.elapsed_time(e) / n


lib = _lib.load()
cases = [(2048, 2048, 921, 921), (2048, 2048, 450, 450), (2048, 2048, 245, 245), (2048, 2048, 143, 143),
         (2160, 3840, 540, 960)]
if len(_sys.argv) > 1:
    cases = [c for c in cases if str(c[2]) in _sys.argv[1:]]
for H, W, oh, ow in cases:
    P = 48
    x = torch.rand((P, H, W), device="cuda").bfloat16()
    ra, ca = _axis.lanczos3(H, oh, 0), _axis.lanczos3(W, ow, 0)
    mid = torch.empty((P, oh, W), dtype=torch.bfloat16, device="cuda")
    owp = -(-ow // 8) * 8
    out = torch.empty((P, oh, owp), dtype=torch.bfloat16, device="cuda")
    st = pipelines._stream(x)
    v = lambda: _lib.check(lib.ts_axis_pass(ra.handle, 0, P, H, W, x.data_ptr(), W, W * H, mid.data_ptr(),
                                            W, W * oh, _lib.TS_BF16, st))
    h = lambda: _lib.check(lib.ts_axis_pass(ca.handle, 1, P, oh, W, mid.data_ptr(), W, W * oh,
                                            out.data_ptr(), owp, owp * oh, _lib.TS_BF16, st))
    tv, th = t(v), t(h)
    tr = t(lambda: pipelines.resample(x, oh, ow))
    vb = P * (H * W + oh * W) * 2
    hb = P * (oh * W + oh * ow) * 2
    print(json.dumps({"cfg": f"{H}x{W}->{oh}x{ow}", "K": [ra.info["window"], ca.info["window"]],
                      "v_ms": round(tv, 4), "v_GBps": round(vb / tv / 1e6), "h_ms": round(th, 4),
                      "h_GBps": round(hb / th / 1e6), "resample_ms": round(tr, 4)}), flush=True)
    del x, mid, out
