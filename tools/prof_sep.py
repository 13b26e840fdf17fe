"""Profiling driver: a few launches of the 4K->1080p Lanczos kernel (8 frames)."""
import os as _os, sys as _sys
_sys.path.insert(0, _os.path.dirname(_os.path.dirname(_os.path.abspath(__file__))))

import sys
import torch
from paper_2512_02371_b200 import pipelines
frames = int(sys.argv[1]) if len(sys.argv) > 1 else 8
x = torch.rand((frames * 3, 2160, 3840), device="cuda").bfloat16()
for _ in range(3):
    y = pipelines.downsample2x(x)
torch.cuda.synchronize()
print("ok", y.shape)
