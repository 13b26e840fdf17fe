import os as _os, sys as _sys
_sys.path.insert(0, _os.path.dirname(_os.path.dirname(_os.path.abspath(__file__))))
import time, torch, json, sys
from paper_2512_02371_b200 import pipelines
def t(fn, x, n=20):
    for _ in range(3): y = fn(x)
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(n): y = fn(x)
    e.record(); torch.cuda.synchronize()
    return s.elapsed_time(e) / n, y
x = torch.rand((8*3, 2160, 3840), device="cuda").bfloat16()
ms, y = t(pipelines.downsample2x, x)
byts = x.numel()*2 + y.numel()*2
print(json.dumps({"cfg": "c2x8", "ms": ms, "GBps": byts/ms/1e6, "Mpix_s": 8*2160*3840/ms/1e3}))
x = torch.rand((3, 2160, 3840), device="cuda").bfloat16()
ms, y = t(pipelines.downsample2x, x)
print(json.dumps({"cfg": "c2x1", "ms": ms, "GBps": (x.numel()*2 + y.numel()*2)/ms/1e6}))
x = torch.rand((3, 4320, 7680), device="cuda").bfloat16()
for taps in (9, 15, 21, 31):
    ms, y = t(lambda z: pipelines.gaussian_blur(z, taps), x)
    print(json.dumps({"cfg": f"c3 gauss{taps}", "ms": ms, "GBps": (x.numel()*2 + y.numel()*2)/ms/1e6}))
x = torch.rand((3, 1080, 1920), device="cuda")
ms, y = t(pipelines.downsample2x, x)
print(json.dumps({"cfg": "c1 f32", "ms": ms, "GBps": (x.numel()*4 + y.numel()*4)/ms/1e6}))
