"""One launch over a large batch vs the same batch as launches of C planes."""
import os, sys, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2512_02371_b200 import pipelines

for F in (48, 128):
    x = torch.rand((3 * F, 2160, 3840), device="cuda").bfloat16()
    out = torch.empty((3 * F, 1080, 1920), device="cuda", dtype=torch.bfloat16)
    for C in (None, 96, 48, 24):
        def step():
            if C is None:
                return pipelines.downsample2x(x)
            for c0 in range(0, 3 * F, C):
                out[c0:c0 + C] = pipelines.downsample2x(x[c0:c0 + C])
        for _ in range(3):
            step()
        torch.cuda.synchronize()
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record()
        for _ in range(10):
            step()
        e.record(); torch.cuda.synchronize()
        ms = s.elapsed_time(e) / 10
        print(json.dumps({"frames": F, "planes_per_launch": C, "ms": round(ms, 4),
                          "ms_per_16_frames": round(ms * 16 / F, 4)}))
    del x, out
