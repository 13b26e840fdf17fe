import os as _os, sys as _sys
_sys.path.insert(0, _os.path.dirname(_os.path.dirname(_os.path.abspath(__file__))))
import json, torch
from paper_2512_02371_b200 import pipelines
def t(fn, n=20):
    for _ in range(3): y = fn()
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(n): y = fn()
    e.record(); torch.cuda.synchronize()
    return s.elapsed_time(e) / n, y
for name, shape, oh, ow in [("4k->540p", (48, 2160, 3840), 540, 960), ("2048->143", (48, 2048, 2048), 143, 143),
                            ("4k->1080p(fused)", (48, 2160, 3840), 1080, 1920)]:
    x = torch.rand(shape, device="cuda").bfloat16()
    ms, y = t(lambda: pipelines.resample(x, oh, ow))
    print(json.dumps({"cfg": name, "ms": round(ms, 4), "in_GBps": round(x.numel() * 2 / ms / 1e6, 1),
                      "Mpix_s": round(shape[0] / 3 * shape[1] * shape[2] / ms / 1e3, 1)}), flush=True)
    del x, y
