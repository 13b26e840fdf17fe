"""Cost of the in-kernel output epilogue (clamp / scale / bias) on config c2
(fused), a two-pass resample and the DCT: plain vs with an epilogue."""
import os as _os, sys as _sys
_sys.path.insert(0, _os.path.dirname(_os.path.dirname(_os.path.abspath(__file__))))
import json, torch
from paper_2512_02371_b200 import pipelines


def t(fn, n=20):
    for _ in range(3): fn()
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(n): fn()
    e.record(); torch.cuda.synchronize()
    return s.elapsed_time(e) / n


x = torch.rand((24, 2160, 3840), device="cuda").bfloat16()
y = torch.rand((48, 2048, 2048), device="cuda").bfloat16()
for name, fn in [("c2x8 resample 2x", lambda **kw: pipelines.downsample2x(x, **kw)),
                 ("2048^2->921^2 two-pass", lambda **kw: pipelines.resample(y, 921, 921, **kw)),
                 ("c4x8 dct16", lambda **kw: pipelines.denoise_dct16(x, 0.15, **kw))]:
    a = t(lambda: fn())
    b = t(lambda: fn(clamp=(0.0, 1.0)))
    print(json.dumps({"cfg": name, "plain_ms": round(a, 4), "clamp_ms": round(b, 4),
                      "overhead": round(b / a - 1, 4)}), flush=True)
