"""Profiling driver: a few launches of the f32 FMA-pipe kernel on config c1
(16 frames of 1080p RGB f32 -> 540p)."""
import os as _os, sys as _sys
_sys.path.insert(0, _os.path.dirname(_os.path.dirname(_os.path.abspath(__file__))))

import torch
from paper_2512_02371_b200 import pipelines
x = torch.rand((48, 1080, 1920), device="cuda")
for _ in range(3):
    y = pipelines.resample(x, 540, 960)
torch.cuda.synchronize()
print("ok", y.shape)
