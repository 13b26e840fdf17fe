import os as _os, sys as _sys
_sys.path.insert(0, _os.path.dirname(_os.path.dirname(_os.path.abspath(__file__))))
import os, json, torch
from paper_2512_02371_b200 import pipelines
def t(fn, n=20):
    for _ in range(3): y = fn()
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(n): y = fn()
    e.record(); torch.cuda.synchronize()
    return s.elapsed_time(e) / n
for name, shape, oh, ow in [("4k->540p", (48, 2160, 3840), 540, 960), ("2048->143", (48, 2048, 2048), 143, 143),
                            ("2048->450", (48, 2048, 2048), 450, 450), ("2048->921", (48, 2048, 2048), 921, 921)]:
    x = torch.rand(shape, device="cuda").bfloat16()
    res = {}
    for nbg in ("auto", "1", "2", "4", "8"):
        if nbg == "auto": os.environ.pop("TSB_APASS_NBG", None)
        else: os.environ["TSB_APASS_NBG"] = nbg
        res[nbg] = round(t(lambda: pipelines.resample(x, oh, ow)), 4)
    print(json.dumps({"cfg": name, "ms": res}), flush=True)
    del x
