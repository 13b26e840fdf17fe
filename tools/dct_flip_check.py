"""Hard-coring flips of the GPU DCT-16 denoise against the oracle: for every
pixel off by > 1e-2, the smallest ||c| - thr| among the coefficients of the
tiles covering it (how close to the threshold the deciding coefficient was).
    python tools/dct_flip_check.py [H W]"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
from oracle import pipelines_ref as R
from paper_2512_02371_b200 import pipelines

H, W = (int(sys.argv[1]), int(sys.argv[2])) if len(sys.argv) > 2 else (232, 360)
rng = np.random.default_rng(3)
yy, xx = np.mgrid[0:H, 0:W]
clean = 0.5 + 0.4 * np.sin(xx / 17.0) * np.cos(yy / 23.0)
x = np.clip(clean + rng.normal(0, 0.05, (1, H, W)), 0, 1).astype(np.float32)
x = torch.from_numpy(x).bfloat16().float().numpy()
y = pipelines.denoise_dct16(torch.from_numpy(x).bfloat16().cuda(), 0.15, "hard",
                            out_dtype=torch.float32).cpu().numpy()
ref = R.dct_denoise(x, 0.15, "hard")
C = R.dct_coefficients(x)
d = np.abs(y - ref)
print("max diff", d.max(), "pixels > 1e-2:", int((d > 1e-2).sum()), "of", d.size)
gap = np.abs(np.abs(C) - np.float32(0.15))
gap[..., 0, 0] = np.inf
tg = gap.min(axis=(-1, -2))[0]  # (ty, tx)
for (p, r, c) in list(zip(*np.nonzero(d > 1e-2)))[:10]:
    ti = [r // 8, r // 8 + 1]
    tj = [c // 8, c // 8 + 1]
    m = min(tg[i, j] for i in ti for j in tj)
    print(f"pixel ({r},{c}) diff {d[p, r, c]:.4f}  closest coefficient gap {m:.3e}")
soft = pipelines.denoise_dct16(torch.from_numpy(x).bfloat16().cuda(), 0.15, "soft",
                               out_dtype=torch.float32).cpu().numpy()
print("soft max diff", np.abs(soft - R.dct_denoise(x, 0.15, "soft")).max())
z = pipelines.denoise_dct16(torch.from_numpy(x).bfloat16().cuda(), 0.0, "soft",
                            out_dtype=torch.float32).cpu().numpy()
print("threshold 0 max diff vs input", np.abs(z - x).max())
