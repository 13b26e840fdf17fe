"""One fused-kernel launch of the 8K Gaussian (config c3), F frames (ncu driver)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2512_02371_b200 import pipelines
taps = int(sys.argv[1]) if len(sys.argv) > 1 else 31
F = int(sys.argv[2]) if len(sys.argv) > 2 else 2
x = torch.rand((3 * F, 4320, 7680), device="cuda").bfloat16()
for _ in range(2):
    y = pipelines.gaussian_blur(x, taps)
torch.cuda.synchronize()
