import os as _os, sys as _sys
_sys.path.insert(0, _os.path.dirname(_os.path.dirname(_os.path.abspath(__file__))))
import os, json, torch
from paper_2512_02371_b200 import pipelines
def t(fn, x, n=30):
    for _ in range(3): y = fn(x)
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(n): y = fn(x)
    e.record(); torch.cuda.synchronize()
    return s.elapsed_time(e) / n, y
cases = [("c2x16", lambda: torch.rand((16*3, 2160, 3840), device="cuda").bfloat16(), pipelines.downsample2x),
         ("up2x", lambda: torch.rand((8*3, 1080, 1920), device="cuda").bfloat16(), pipelines.upsample2x)]
for taps in (9, 15, 21, 31):
    cases.append((f"gauss{taps}", lambda: torch.rand((3, 4320, 7680), device="cuda").bfloat16(),
                  (lambda tp: (lambda z: pipelines.gaussian_blur(z, tp)))(taps)))
for name, mk, fn in cases:
    x = mk()
    for v in ("5", "4"):
        if v == "5": os.environ["TSB_STRIP"] = "1"
        else: os.environ.pop("TSB_STRIP", None)
        ms, y = t(fn, x)
        print(json.dumps({"cfg": name, "v": v, "ms": round(ms, 4), "GBps": round((x.numel()*2 + y.numel()*2)/ms/1e6, 1)}), flush=True)
    del x, y
