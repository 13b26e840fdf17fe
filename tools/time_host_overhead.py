import os as _os, sys as _sys
_sys.path.insert(0, _os.path.dirname(_os.path.dirname(_os.path.abspath(__file__))))
import time, json, torch
from paper_2512_02371_b200 import pipelines
x = torch.rand((3, 1080, 1920), device="cuda").bfloat16()
x4 = torch.rand((3, 2160, 3840), device="cuda").bfloat16()
for name, fn in (("1080p->540p bf16", lambda: pipelines.downsample2x(x)),
                 ("4K->1080p bf16", lambda: pipelines.downsample2x(x4)),
                 ("4K dct16", lambda: pipelines.denoise_dct16(x4, 0.15))):
    for _ in range(20): fn()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(200): fn()
    t1 = time.perf_counter()
    torch.cuda.synchronize()
    t2 = time.perf_counter()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record(); fn(); e.record(); torch.cuda.synchronize()
    print(json.dumps({"case": name, "host_us_per_call": round((t1 - t0) / 200 * 1e6, 1),
                      "wall_us_per_call": round((t2 - t0) / 200 * 1e6, 1), "device_us": round(s.elapsed_time(e) * 1e3, 1)}))
