"""f32 images through the FMA-pipe kernel (csrc/separable_f32.cu).

The kernel evaluates the reference's two source-form conv passes in their
exact order (horizontal first, f32 products summed left to right, + 0;
interp.py:162-167, 203-211, restated in oracle/pipelines_ref.py:78-97), so
in exact mode (pipelines.F32_EXACT / TSB_F32_EXACT=1) its f32 output must
equal the oracle's BIT FOR BIT — no tolerance; the default fused-multiply-add
mode differs by f32 rounding only (bound 1e-6 on [0,1] images).
"""

import numpy as np
import pytest

from oracle import pipelines_ref as ref


def _torch():
    import torch
    return torch


def _img(shape, seed):
    return np.random.default_rng(seed).random(shape, dtype=np.float32)


def test_filters_weights_match_oracle_bitwise():
    """The host taps the f32 kernel uploads are the oracle's, bit for bit."""
    from paper_2512_02371_b200 import filters
    for n_in, n_out in ((1080, 540), (1920, 960), (271, 135), (7, 3), (2160, 1080)):
        f0, w0 = filters.lanczos3_axis(n_in, n_out)
        f1, w1 = ref.lanczos3_weights(n_in, n_out)
        assert np.array_equal(np.asarray(f0, np.int64), f1)
        assert np.array_equal(np.asarray(w0, np.float32), w1)
    for taps in (9, 15, 21, 31):
        k0 = filters.gaussian_taps(taps)
        assert np.array_equal(np.asarray(k0, np.float32), ref.gaussian_kernel(taps))


def test_uniform_axis_detection():
    from paper_2512_02371_b200 import axis, filters
    pytest.importorskip("torch")
    # host-side property only (no device work): build the tables without a handle
    a = axis.Axis.__new__(axis.Axis)
    a.n_out = 540
    a.first, a.weights = filters.lanczos3_axis(1080, 540)
    assert a.uniform == (2, 12, -5)
    a.n_out = 135
    a.first, a.weights = filters.lanczos3_axis(2048, 135)  # non-integer factor
    assert a.uniform is None or a.uniform[0] != 2 or a.uniform[1] != 12


@pytest.mark.gpu
@pytest.mark.parametrize("shape,oh,ow", [
    ((3, 1080, 1920), 540, 960),     # config c1
    ((3, 270, 482), 135, 241),       # ragged tiles on both axes
    ((1, 8, 12), 4, 6),              # image smaller than one window
    ((2, 3, 64, 128), 32, 64),       # leading batch dims
])
def test_lanczos2x_f32_bitexact(shape, oh, ow, monkeypatch):
    torch = _torch()
    from paper_2512_02371_b200 import pipelines
    x = _img(shape, 11)
    want = ref.resample(x, oh, ow)
    fast = pipelines.resample(torch.from_numpy(x).cuda(), oh, ow, out_dtype=torch.float32)
    assert np.abs(fast.cpu().numpy() - want).max() <= 1e-6
    monkeypatch.setattr(pipelines, "F32_EXACT", True)
    y = pipelines.resample(torch.from_numpy(x).cuda(), oh, ow, out_dtype=torch.float32)
    torch.cuda.synchronize()
    got = y.cpu().numpy()
    assert got.shape == want.shape
    assert np.array_equal(got.view(np.uint32), want.view(np.uint32)), \
        f"{np.count_nonzero(got != want)} pixels differ, max {np.abs(got - want).max()}"


@pytest.mark.gpu
@pytest.mark.parametrize("taps", [9, 15, 21, 31])
def test_gaussian_f32_bitexact(taps, monkeypatch):
    torch = _torch()
    from paper_2512_02371_b200 import pipelines
    x = _img((2, 200, 333), taps)
    fast = pipelines.gaussian_blur(torch.from_numpy(x).cuda(), taps, out_dtype=torch.float32)
    assert np.abs(fast.cpu().numpy() - ref.gaussian_blur(x, taps)).max() <= 1e-6
    monkeypatch.setattr(pipelines, "F32_EXACT", True)
    y = pipelines.gaussian_blur(torch.from_numpy(x).cuda(), taps, out_dtype=torch.float32)
    torch.cuda.synchronize()
    want = ref.gaussian_blur(x, taps)
    assert np.array_equal(y.cpu().numpy().view(np.uint32), want.view(np.uint32))


@pytest.mark.gpu
def test_f32_bf16_out_and_epilogue():
    """bf16 output = RNE of the f32 output; the epilogue = clamp(scale·y + bias)
    of the plain output (fmaf, as the tensor-core kernels apply it)."""
    torch = _torch()
    from paper_2512_02371_b200 import pipelines
    x = torch.from_numpy(_img((3, 270, 480), 5) * 1.4 - 0.2).cuda()
    y32 = pipelines.downsample2x(x, out_dtype=torch.float32)
    y16 = pipelines.downsample2x(x, out_dtype=torch.bfloat16)
    assert torch.equal(y16, y32.bfloat16())
    ye = pipelines.downsample2x(x, out_dtype=torch.float32, clamp=(0.0, 1.0), scale=0.5,
                                bias=0.25)
    want = torch.clamp(torch.addcmul(torch.full_like(y32, 0.25), y32, torch.full_like(y32, 0.5)),
                       0.0, 1.0)
    assert (ye - want).abs().max().item() <= 1e-7
    yb = pipelines.downsample2x(x, out_dtype=torch.bfloat16, clamp=(0.0, 1.0))
    assert torch.equal(yb, torch.clamp(y32, 0.0, 1.0).bfloat16())


@pytest.mark.gpu
def test_f32_kernel_is_the_one_launched():
    """f32 inputs take ts_separable_f32_ep (no bf16 copy), bf16 inputs do not."""
    torch = _torch()
    from paper_2512_02371_b200 import axis, pipelines
    dev = torch.cuda.current_device()
    ra, ca = axis.lanczos3(64, 32, dev), axis.lanczos3(128, 64, dev)
    x = torch.rand((1, 64, 128), device="cuda")
    assert pipelines._run_f32(x, ra, ca, torch.float32, None, pipelines._stream(x)) is not None
    # non-uniform axes (non-integer factor) fall through to the tensor-core path
    rb = axis.lanczos3(64, 27, dev)
    if rb.uniform is None:
        assert pipelines._run_f32(x, rb, ca, torch.float32, None, pipelines._stream(x)) is None


@pytest.mark.gpu
def test_unsupported_out_dtype_raises():
    """An out dtype the kernels cannot write is rejected before any launch."""
    torch = _torch()
    from paper_2512_02371_b200 import pipelines
    for x in (torch.rand((1, 64, 128), device="cuda"),
              torch.rand((1, 64, 128), device="cuda").bfloat16()):
        with pytest.raises(TypeError):
            pipelines.downsample2x(x, out_dtype=torch.float16)
