"""Fraction of pixels where GPU hard coring differs from the oracle by more
than 1e-2 (threshold ties), per band-width variant."""
import os as _os, sys as _sys
_sys.path.insert(0, _os.path.dirname(_os.path.dirname(_os.path.abspath(__file__))))
import json, os
import numpy as np, torch
from oracle import pipelines_ref
from paper_2512_02371_b200 import pipelines
rng = np.random.default_rng(3)
H, W = 1080, 1920
yy, xx = np.mgrid[0:H, 0:W]
clean = 0.5 + 0.4 * np.sin(xx / 17.0) * np.cos(yy / 23.0)
x = np.clip(clean + rng.normal(0, 0.05, (1, H, W)), 0, 1).astype(np.float32)
x = torch.from_numpy(x).bfloat16().float().numpy()
ref = pipelines_ref.dct_denoise(x, 0.15, "hard")
for bw in ("64", "128"):
    os.environ["TSB_DCT_BAND"] = bw
    y = pipelines.denoise_dct16(torch.from_numpy(x).bfloat16().cuda(), 0.15, "hard",
                                out_dtype=torch.float32).cpu().numpy()
    d = np.abs(y - ref)
    print(json.dumps({"band": bw, "frac_gt_1e-2": float((d > 1e-2).mean()), "max": float(d.max()),
                      "p99.99": float(np.quantile(d, 0.9999))}))
