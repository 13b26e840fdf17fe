"""GPU parity of the fused separable kernel and the tcgen05 layout probe.

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


def test_probe_umma_layouts():
    torch = _torch()
    from paper_2512_02371_b200 import _lib
    g = torch.Generator(device="cpu").manual_seed(0)
    for k, n in ((16, 16), (48, 16), (64, 32), (128, 128), (256, 256)):
        a = torch.randn(128, k, generator=g).bfloat16().float().cuda()
        b = torch.randn(k, n, generator=g).bfloat16().float().cuda()
        d = torch.zeros(128, n, device="cuda")
        _lib.check(_lib.load().ts_probe_umma(a.data_ptr(), b.data_ptr(), d.data_ptr(), k, n,
                                             torch.cuda.current_stream().cuda_stream))
        torch.cuda.synchronize()
        ref = a @ b
        err = (d - ref).abs().max().item()
        assert err < 1e-3 * max(1.0, ref.abs().max().item()), (k, n, err)


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


def _variant(ra, ca, planes=1, out_dtype=1):
    from paper_2512_02371_b200 import _lib
    return _lib.load().ts_separable_variant(ra.handle, ca.handle, planes, out_dtype)


@pytest.mark.parametrize("case", [
    ("down", (3, 2160, 3840)), ("down", (1, 1080, 1920)), ("down", (2, 300, 200)),
    ("down", (1, 264, 392)), ("up", (3, 135, 240)), ("gauss9", (3, 200, 328)),
    ("gauss31", (3, 544, 1000)), ("box5", (2, 256, 520)),
])
def test_strip_kernel_matches_block_kernel(case, monkeypatch):
    """The strip kernel (Toeplitz-like axes, opt-in via TSB_STRIP=1) against
    the block-tile kernel on the same bf16 weights: identical up to
    intermediate rounding."""
    torch = _torch()
    from paper_2512_02371_b200 import pipelines
    kind, shape = case
    g = torch.Generator(device="cpu").manual_seed(sum(shape))
    x = torch.rand(shape, generator=g).bfloat16().cuda()
    if kind == "down":
        fn = lambda: pipelines.downsample2x(x, out_dtype=torch.float32)
    elif kind == "up":
        fn = lambda: pipelines.upsample2x(x, out_dtype=torch.float32)
    elif kind.startswith("gauss"):
        fn = lambda: pipelines.gaussian_blur(x, int(kind[5:]), out_dtype=torch.float32)
    else:
        fn = lambda: pipelines.box_blur(x, int(kind[3:]), out_dtype=torch.float32)
    monkeypatch.setenv("TSB_STRIP", "1")
    y5 = fn()
    monkeypatch.delenv("TSB_STRIP")
    y4 = fn()
    torch.cuda.synchronize()
    assert y5.shape == y4.shape
    d = (y5 - y4).abs()
    # different f32 summation order -> rare 1-ulp flips of the bf16 intermediate
    assert d.max().item() <= 2e-3, d.max().item()
    assert (d > 1e-5).float().mean().item() < 0.05


def test_strip_variant_selection(monkeypatch):
    from paper_2512_02371_b200 import axis, filters
    lz = axis.lanczos3(2160, 1080, 0), axis.lanczos3(3840, 1920, 0)
    monkeypatch.delenv("TSB_STRIP", raising=False)
    assert _variant(*lz, 3) == 4
    monkeypatch.setenv("TSB_STRIP", "1")
    lz = axis.lanczos3(2160, 1080, 0), axis.lanczos3(3840, 1920, 0)
    assert _variant(*lz, 3) == 5
    odd = axis.lanczos3(1080, 720, 0), axis.lanczos3(1920, 1280, 0)
    assert _variant(*odd, 3) == 4
    k = filters.gaussian_taps(9)
    assert _variant(axis.convolution(512, k, 0), axis.convolution(1024, k, 0)) == 5

