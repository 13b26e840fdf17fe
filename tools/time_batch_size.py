"""Per-frame cost of the fused c2 kernel vs batch size and working set:
launches of F frames over NB distinct input buffers (round-robin)."""
import os, sys, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2512_02371_b200 import pipelines

def run(F, NB, reps=40):
    xs = [torch.rand((3 * F, 2160, 3840), device="cuda").bfloat16() for _ in range(NB)]
    for i in range(5):
        pipelines.downsample2x(xs[i % NB])
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for i in range(reps):
        pipelines.downsample2x(xs[i % NB])
    e.record(); torch.cuda.synchronize()
    ms = s.elapsed_time(e) / reps
    del xs
    torch.cuda.empty_cache()
    return ms

for F, NB in ((16, 2), (16, 6), (16, 12), (48, 1), (48, 2), (8, 2), (8, 12), (4, 24)):
    ms = run(F, NB)
    print(json.dumps({"frames": F, "buffers": NB, "ms": round(ms, 4),
                      "ms_per_16_frames": round(ms * 16 / F, 4),
                      "working_set_GB": round(NB * 3 * F * 2160 * 3840 * 2 / 1e9, 2)}))
