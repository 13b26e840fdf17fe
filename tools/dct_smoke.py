"""Tiny DCT-16 runs of increasing size against the oracle (debug driver)."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
from oracle import pipelines_ref as R
from paper_2512_02371_b200 import pipelines
for shape in [(1, 16, 16), (1, 64, 48), (1, 72, 48), (1, 136, 96), (2, 232, 360)]:
    x = torch.rand(shape).bfloat16()
    t = time.time()
    y = pipelines.denoise_dct16(x.cuda(), 0.0, "soft", out_dtype=torch.float32)
    torch.cuda.synchronize()
    err = np.abs(y.cpu().numpy() - x.float().numpy()).max()
    ref = R.dct_denoise(x.float().numpy(), 0.15, "soft")
    y2 = pipelines.denoise_dct16(x.cuda(), 0.15, "soft", out_dtype=torch.float32).cpu().numpy()
    print(shape, "identity err", err, "soft err", np.abs(y2 - ref).max(), f"{time.time() - t:.2f}s", flush=True)
