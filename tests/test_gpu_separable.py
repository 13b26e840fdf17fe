"""GPU parity of the fused separable kernel.

Kernel-level checks compare against a plain PyTorch fp32 emulation of the
same arithmetic (bf16 operands, f32 accumulate, bf16 intermediate) using the
effective weights the builder produced (Axis.dense()); image-level parity
against the CPU oracle lives in test_gpu_parity.py.
"""

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _torch():
    import torch
    return torch


def _emulate(x, R, C, out_dtype):
    """fp32 emulation of the kernel: V = bf16(R @ X); out = cast(V @ Cᵀ)."""
    torch = _torch()
    R = torch.as_tensor(R, device=x.device)
    C = torch.as_tensor(C, device=x.device)
    xf = x.float()
    v = torch.matmul(R, xf).bfloat16().float()
    out = torch.matmul(v, C.t())
    return out.to(out_dtype)


@pytest.mark.parametrize("shape,oshape", [
    ((1, 64, 64), (32, 32)),
    ((3, 270, 480), (135, 240)),
    ((2, 300, 200), (150, 100)),
    ((1, 1080, 1920), (540, 960)),
    ((3, 2160, 3840), (1080, 1920)),
])
def test_lanczos_kernel_matches_emulation(shape, oshape):
    torch = _torch()
    from paper_2512_02371_b200 import axis, pipelines
    g = torch.Generator(device="cpu").manual_seed(1)
    x = torch.rand(shape, generator=g).bfloat16().cuda()
    y = pipelines.resample(x, *oshape)
    torch.cuda.synchronize()
    R = axis.lanczos3(shape[-2], oshape[0], 0).dense()
    C = axis.lanczos3(shape[-1], oshape[1], 0).dense()
    ref = _emulate(x, R, C, torch.float32)
    err = (y.float() - ref).abs().max().item()
    assert y.shape == (shape[0],) + tuple(oshape)
    # bf16 output rounding (half ulp of values <= ~1.2) + f32 summation order
    assert err <= 4e-3, err


@pytest.mark.parametrize("taps", [9, 15, 21, 31])
def test_gaussian_kernel_matches_emulation(taps):
    torch = _torch()
    from paper_2512_02371_b200 import axis, filters, pipelines
    g = torch.Generator(device="cpu").manual_seed(taps)
    x = torch.rand((3, 200, 328), generator=g).bfloat16().cuda()
    y = pipelines.gaussian_blur(x, taps, out_dtype=torch.float32)
    torch.cuda.synchronize()
    k = filters.gaussian_taps(taps)
    R = axis.convolution(200, k, 0).dense()
    C = axis.convolution(328, k, 0).dense()
    ref = _emulate(x, R, C, torch.float32)
    err = (y - ref).abs().max().item()
    # one bf16 ulp flip of the intermediate (sum-order differences) times a tap
    assert err <= 2e-3, err


def test_f32_input_and_output():
    torch = _torch()
    from paper_2512_02371_b200 import pipelines
    g = torch.Generator(device="cpu").manual_seed(3)
    x = torch.rand((3, 1080, 1920), generator=g).cuda()
    y = pipelines.downsample2x(x)
    assert y.dtype == torch.float32 and y.shape == (3, 540, 960)
    # f32 images take the f32 FMA-pipe kernel (test_gpu_separable_f32.py);
    # the bf16 tensor-core path differs from it by bf16 operand rounding
    yb = pipelines.downsample2x(x.bfloat16(), out_dtype=torch.float32)
    torch.cuda.synchronize()
    assert (y - yb).abs().max().item() <= 8e-3


def test_end_of_work_signals_never_run_two_phases_ahead():
    """Regression (found by tools/fuzz_pipelines.py): a plan with one V
    buffer (3 x 906 x 1374, 3 / 19-tap Gaussians, f32 out: merged axes, 48 KB
    of f32 staging) where CTAs process three tiles.  The end-of-work
    sentinel used to pass each hand-off barrier without waiting for its
    'free' twin, so with a slow epilogue a barrier completed two phases
    before its waiter looked and the waiter's parity test blocked forever
    (the mbarrier watchdog turned it into a launch failure after 4 s).  Run
    in a subprocess: a hang must not take this test process's context."""
    import os
    import subprocess
    import sys
    code = r"""
import torch
from paper_2512_02371_b200 import filters, pipelines
from oracle import pipelines_ref
import numpy as np
g = torch.Generator(device="cpu").manual_seed(3)
x = torch.rand((3, 906, 1374), generator=g).bfloat16()
kv, kh = filters.gaussian_taps(3), filters.gaussian_taps(19)
for od in (torch.float32, torch.bfloat16):
    y = pipelines.filter_separable(x.cuda(), kv, kh, out_dtype=od).float().cpu().numpy()
    ref = pipelines_ref.separable(x.float().numpy(), pipelines_ref.centred_axis(906, kv),
                                  pipelines_ref.centred_axis(1374, kh))
    assert np.abs(y - ref).max() <= 1e-2
print("ok")
"""
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    r = subprocess.run([sys.executable, "-c", code], capture_output=True, text=True, timeout=300,
                       cwd=root)
    assert r.returncode == 0 and r.stdout.strip().endswith("ok"), r.stdout + r.stderr
