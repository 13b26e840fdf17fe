"""One fused-kernel launch over F frames (ncu driver)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2512_02371_b200 import pipelines
F = int(sys.argv[1]) if len(sys.argv) > 1 else 16
x = torch.rand((3 * F, 2160, 3840), device="cuda").bfloat16()
for _ in range(2):
    y = pipelines.downsample2x(x)
torch.cuda.synchronize()
