import os as _os, sys as _sys
_sys.path.insert(0, _os.path.dirname(_os.path.dirname(_os.path.abspath(__file__))))
import torch, json, sys
from paper_2512_02371_b200 import pipelines
F = int(sys.argv[1]) if len(sys.argv) > 1 else 4
x = torch.rand((3 * F, 2160, 3840), device="cuda").bfloat16()
for _ in range(3): y = pipelines.denoise_dct16(x, 0.15)
torch.cuda.synchronize()
s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
s.record()
for _ in range(10): y = pipelines.denoise_dct16(x, 0.15)
e.record(); torch.cuda.synchronize()
ms = s.elapsed_time(e) / 10
print(json.dumps({"cfg": f"c4 x{F} frames", "ms": ms, "ms_per_frame": ms / F, "GBps": (x.numel() * 4) / ms / 1e6, "Mpix_s": F * 2160 * 3840 / ms / 1e3}))
