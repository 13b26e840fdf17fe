"""Seeded random geometries through the public pipelines against the CPU
oracle: image sizes from a few pixels to ~1500, up- and downscale factors
from 0.5x to ~40x per axis independently (so both the fused kernel and the
persistent axis passes run, with ragged strips, short last groups and
one-block axes), Gaussian widths 3-61 taps, bf16 and f32 outputs.  Same
tolerance as the parity tests (max |gpu - oracle| <= 1e-2 on [0, 1]
images).  Reference semantics: the separable pipelines of PAPER.md:950-979
evaluated by interp.run_program's tile loop (interp.py:570-619)."""

import numpy as np
import pytest

from oracle import pipelines_ref

pytestmark = pytest.mark.gpu
TOL = 1e-2


def _cases(n, seed):
    rng = np.random.default_rng(seed)
    out = []
    for _ in range(n):
        H = int(rng.integers(8, 1500))
        W = int(rng.integers(8, 1500))
        # per-axis factor: log-uniform in [1/2, 40], at least one output
        fh, fw = np.exp(rng.uniform(np.log(0.5), np.log(40.0), 2))
        oh = max(1, min(3000, int(round(H / fh))))
        ow = max(1, min(3000, int(round(W / fw))))
        planes = int(rng.integers(1, 4))
        f32 = bool(rng.integers(0, 2))
        out.append((planes, H, W, oh, ow, f32))
    return out


@pytest.mark.parametrize("planes,H,W,oh,ow,f32", _cases(24, 2512))
def test_random_resample_matches_oracle(planes, H, W, oh, ow, f32):
    import torch
    from paper_2512_02371_b200 import pipelines
    rng = np.random.default_rng(H * 7919 + W)
    x = torch.from_numpy(rng.random((planes, H, W), dtype=np.float32)).bfloat16()
    y = pipelines.resample(x.cuda(), oh, ow,
                           out_dtype=torch.float32 if f32 else torch.bfloat16)
    torch.cuda.synchronize()
    assert tuple(y.shape) == (planes, oh, ow)
    ref = pipelines_ref.resample(x.float().numpy(), oh, ow)
    d = np.abs(y.float().cpu().numpy() - ref).max()
    assert d <= TOL, (d, planes, H, W, oh, ow)


def _gauss_cases(n, seed):
    rng = np.random.default_rng(seed)
    return [(int(rng.integers(1, 3)), int(rng.integers(8, 1200)), int(rng.integers(8, 1200)),
             int(2 * rng.integers(1, 31) + 1)) for _ in range(n)]


@pytest.mark.parametrize("planes,H,W,taps", _gauss_cases(12, 31))
def test_random_gaussian_matches_oracle(planes, H, W, taps):
    import torch
    from paper_2512_02371_b200 import pipelines
    rng = np.random.default_rng(taps * 131 + H)
    x = torch.from_numpy(rng.random((planes, H, W), dtype=np.float32)).bfloat16()
    y = pipelines.gaussian_blur(x.cuda(), taps, out_dtype=torch.float32)
    torch.cuda.synchronize()
    ref = pipelines_ref.gaussian_blur(x.float().numpy(), taps)
    d = np.abs(y.cpu().numpy() - ref).max()
    assert d <= TOL, (d, planes, H, W, taps)


def _dct_cases(n, seed):
    rng = np.random.default_rng(seed)
    return [(int(rng.integers(1, 4)), 8 * int(rng.integers(2, 90)), 8 * int(rng.integers(2, 90)),
             float(rng.uniform(0.02, 0.3))) for _ in range(n)]


@pytest.mark.parametrize("planes,H,W,thr", _dct_cases(10, 16))
def test_random_dct16_soft_matches_oracle(planes, H, W, thr):
    """Soft coring (Lipschitz: every pixel within 1e-2) at random sizes —
    strips, segments and the 56-row first-group store on ragged images."""
    import torch
    from paper_2512_02371_b200 import pipelines
    rng = np.random.default_rng(H * 31 + W)
    x = torch.from_numpy(rng.random((planes, H, W), dtype=np.float32)).bfloat16()
    y = pipelines.denoise_dct16(x.cuda(), thr, "soft", out_dtype=torch.float32)
    torch.cuda.synchronize()
    ref = pipelines_ref.dct_denoise(x.float().numpy(), thr, "soft")
    d = np.abs(y.cpu().numpy() - ref).max()
    assert d <= TOL, (d, planes, H, W, thr)
