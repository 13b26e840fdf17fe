#!/bin/bash
# same-box A/B of the fused kernel's per-frame cost at 16 and 48 frames per launch
python - <<'PY'
import os, sys, json
sys.path.insert(0, ".")
import torch
from paper_2512_02371_b200 import pipelines
res = []
for F in (16, 48):
    xs = [torch.rand((3 * F, 2160, 3840), device="cuda").bfloat16() for _ in range(2)]
    for i in range(5):
        pipelines.downsample2x(xs[i % 2])
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for i in range(40):
        pipelines.downsample2x(xs[i % 2])
    e.record(); torch.cuda.synchronize()
    res.append(round(s.elapsed_time(e) / 40 * 16 / F, 4))
    del xs
print("ms per 16 frames at 16 / 48 frames per launch:", res)
PY
