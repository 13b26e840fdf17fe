"""Edge cases of the GPU pipelines against the CPU oracle: empty batches,
tiny and ragged images, degenerate kernels, batched leading dims."""

import numpy as np
import pytest

from oracle import pipelines_ref

pytestmark = pytest.mark.gpu
TOL = 1e-2


def _img(shape, seed):
    import torch
    x = np.random.default_rng(seed).random(shape, dtype=np.float32)
    return torch.from_numpy(x).bfloat16().float().numpy()


def _gpu(fn, x, **kw):
    import torch
    y = fn(torch.from_numpy(x).bfloat16().cuda(), out_dtype=torch.float32, **kw)
    torch.cuda.synchronize()
    return y.cpu().numpy()


def test_empty_batch_returns_empty():
    import torch
    from paper_2512_02371_b200 import pipelines
    x = torch.empty((0, 3, 64, 64), dtype=torch.bfloat16, device="cuda")
    assert pipelines.resample(x, 32, 32).shape == (0, 3, 32, 32)
    assert pipelines.gaussian_blur(x, 9).shape == (0, 3, 64, 64)
    assert pipelines.denoise_dct16(x, 0.1).shape == (0, 3, 64, 64)


@pytest.mark.parametrize("shape,oh,ow", [
    ((1, 1, 1), 1, 1), ((1, 1, 7), 1, 3), ((2, 3, 5), 6, 10), ((1, 9, 1), 4, 1),
    ((1, 17, 33), 8, 16),
])
def test_tiny_and_ragged_resample(shape, oh, ow):
    from paper_2512_02371_b200 import pipelines
    x = _img(shape, 31)
    y = _gpu(pipelines.resample, x, out_h=oh, out_w=ow)
    ref = pipelines_ref.resample(x, oh, ow)
    assert y.shape == ref.shape
    assert np.abs(y - ref).max() <= TOL


def test_batched_leading_dims_match_flat():
    import torch
    from paper_2512_02371_b200 import pipelines
    x = torch.from_numpy(_img((2, 3, 3, 48, 80), 32)).bfloat16().cuda()
    y = pipelines.downsample2x(x, out_dtype=torch.float32)
    yf = pipelines.downsample2x(x.reshape(18, 48, 80), out_dtype=torch.float32)
    assert y.shape == (2, 3, 3, 24, 40)
    assert torch.equal(y.reshape(18, 24, 40), yf)


@pytest.mark.parametrize("taps", [1, 3])
def test_degenerate_gaussian(taps):
    from paper_2512_02371_b200 import pipelines
    x = _img((1, 40, 56), 33)
    y = _gpu(pipelines.gaussian_blur, x, taps=taps)
    ref = pipelines_ref.gaussian_blur(x, taps)
    assert np.abs(y - ref).max() <= TOL
    if taps == 1:
        assert np.abs(y - x).max() <= 4e-3  # identity up to bf16 rounding


@pytest.mark.parametrize("shape", [(1, 8, 8), (1, 8, 24), (2, 40, 8), (1, 120, 232)])
def test_dct_small_and_band_edge_sizes(shape):
    from paper_2512_02371_b200 import pipelines
    x = _img(shape, 34)
    y = _gpu(pipelines.denoise_dct16, x, threshold=0.15, mode="soft")
    ref = pipelines_ref.dct_denoise(x, 0.15, "soft")
    assert np.abs(y - ref).max() <= TOL


def test_f32_output_odd_width():
    from paper_2512_02371_b200 import pipelines
    x = _img((3, 50, 77), 35)
    y = _gpu(pipelines.resample, x, out_h=25, out_w=39)
    ref = pipelines_ref.resample(x, 25, 39)
    assert np.abs(y - ref).max() <= TOL


def test_run_from_host_matches_device_path():
    import torch
    from paper_2512_02371_b200 import pipelines
    x = torch.rand((30, 96, 160)).bfloat16().pin_memory()
    out = torch.empty((30, 48, 80), dtype=torch.bfloat16).pin_memory()
    pipelines.run_from_host(pipelines.downsample2x, x, out, chunk_planes=4, lanes=3)
    torch.cuda.synchronize()
    ref = pipelines.downsample2x(x.cuda()).cpu()
    assert torch.equal(out, ref)


def test_very_long_axis():
    """A 128K-wide axis: beyond the fused kernel's packed block tables (32K
    inputs), so it runs as axis passes (plain ws / tid tables)."""
    from paper_2512_02371_b200 import pipelines
    x = _img((1, 16, 131072), 36)
    y = _gpu(pipelines.resample, x, out_h=8, out_w=65536)
    ref = pipelines_ref.resample(x, 8, 65536)
    assert np.abs(y - ref).max() <= TOL


def test_non_contiguous_and_f32_inputs():
    import torch
    from paper_2512_02371_b200 import pipelines
    base = torch.from_numpy(_img((3, 96, 256), 37)).cuda()
    x = base[:, :, ::2]  # non-contiguous view, 96 x 128
    y = pipelines.downsample2x(x, out_dtype=torch.float32)
    ref = pipelines_ref.resample(x.cpu().contiguous().numpy(), 48, 64)
    assert np.abs(y.cpu().numpy() - ref).max() <= TOL
    with pytest.raises(TypeError):
        pipelines.downsample2x(torch.zeros((1, 16, 16), dtype=torch.int32, device="cuda"))


def test_fused_kernel_global_block_tables():
    """> 3072 block-table entries (rows + columns) but < 32K inputs: the fused
    kernel reads its tables from global memory instead of the parameter bank."""
    from paper_2512_02371_b200 import axis, pipelines
    ra, ca = axis.lanczos3(24000, 48000, 0), axis.lanczos3(48, 96, 0)  # 2x up: 3000+ blocks
    assert ra.info["blocks"] + ca.info["blocks"] + 128 > 3072 and pipelines.fused_supported(ra, ca)
    x = _img((1, 24000, 48), 38)
    y = _gpu(pipelines.resample, x, out_h=48000, out_w=96)
    ref = pipelines_ref.resample(x, 48000, 96)
    assert np.abs(y - ref).max() <= TOL


@pytest.mark.parametrize("case", ["fused", "two_pass", "gauss", "dct"])
def test_output_epilogue_clamp_and_normalise(case):
    """The in-kernel output epilogue (ts_epilogue): clamp / scale / bias
    applied to the f32 result before the cast equal the same operations on
    the plain kernel's f32 output (bitwise for the clamp, f32 rounding of
    one fused multiply-add for scale / bias).  bf16 outputs clamp the packed
    pair against bf16-rounded bounds, which must equal clamping in f32 and
    then rounding, bit for bit; NaN inputs stay NaN through the clamp."""
    import torch
    from paper_2512_02371_b200 import pipelines
    g = torch.Generator(device="cuda").manual_seed(9)
    x = torch.rand((3, 544, 960), device="cuda", generator=g).bfloat16()
    x = x * 1.6 - 0.3  # overshoot both clamp bounds
    fns = {"fused": lambda **kw: pipelines.resample(x, 272, 480, **kw),
           "two_pass": lambda **kw: pipelines.resample(x, 40, 70, **kw),
           "gauss": lambda **kw: pipelines.gaussian_blur(x, 9, **kw),
           "dct": lambda **kw: pipelines.denoise_dct16(x, 0.15, **kw)}
    fn = fns[case]
    f32 = torch.float32
    y = fn(out_dtype=f32)
    yc = fn(out_dtype=f32, clamp=(0.1, 0.9))
    assert torch.equal(yc, y.clamp(0.1, 0.9))
    ys = fn(out_dtype=f32, scale=255.0, bias=-3.0)
    assert torch.allclose(ys, y * 255.0 - 3.0, rtol=1e-6, atol=1e-4)
    yb = fn(out_dtype=f32, scale=2.0, clamp=(0.0, 1.0))
    assert torch.allclose(yb, (y * 2.0).clamp(0.0, 1.0), rtol=1e-6, atol=1e-6)
    # bf16 output: the clamp on the rounded pair == round(clamp in f32)
    for lo, hi in [(0.0, 1.0), (0.1, 0.9), (0.3337, 0.6663)]:
        yh = fn(clamp=(lo, hi))
        assert torch.equal(yh, y.clamp(lo, hi).bfloat16()), (lo, hi)
    yh = fn(scale=2.0, bias=0.25, clamp=(0.0, 1.0))
    assert torch.equal(yh, torch.addcmul(torch.full_like(y, 0.25), y, torch.full_like(y, 2.0))
                       .clamp(0.0, 1.0).bfloat16())
    # NaN propagates through the clamp (both output dtypes)
    xn = x.clone()
    xn[0, 100:140, 200:260] = float("nan")
    fnn = {"fused": lambda **kw: pipelines.resample(xn, 272, 480, **kw),
           "two_pass": lambda **kw: pipelines.resample(xn, 40, 70, **kw),
           "gauss": lambda **kw: pipelines.gaussian_blur(xn, 9, **kw),
           "dct": lambda **kw: pipelines.denoise_dct16(xn, 0.15, **kw)}[case]
    for dt in (f32, torch.bfloat16):
        a = fnn(out_dtype=dt)
        b = fnn(out_dtype=dt, clamp=(0.0, 1.0))
        assert torch.equal(torch.isnan(a), torch.isnan(b))
        assert torch.isnan(b).any()


def test_f32_kernel_more_planes_than_a_grid_dimension():
    """70000 tiny f32 planes (> 65535, the old grid.z limit): the persistent
    f32 kernel walks them all, bit-exact in exact mode."""
    import torch
    from paper_2512_02371_b200 import pipelines
    x = torch.from_numpy(np.random.default_rng(38).random((70000, 8, 16), dtype=np.float32))
    exact, pipelines.F32_EXACT = pipelines.F32_EXACT, True
    try:
        y = pipelines.resample(x.cuda(), 4, 8, out_dtype=torch.float32)
        torch.cuda.synchronize()
    finally:
        pipelines.F32_EXACT = exact
    ref = pipelines_ref.resample(x.numpy(), 4, 8)
    assert np.array_equal(y.cpu().numpy().view(np.uint32), ref.view(np.uint32))


@pytest.mark.parametrize("shape,oh,ow", [
    ((1, 64, 40000), 32, 20000),    # columns past the fused kernel's packed +-32K tables
    ((1, 40000, 64), 20000, 32),    # rows likewise
    ((1, 70000, 48), 3000, 48),     # a 23x row factor on a very tall image
    ((1, 16384, 16384), 1000, 1000),  # 512 MB plane through the axis passes
])
def test_extreme_image_sizes_match_oracle(shape, oh, ow):
    import numpy as np
    import torch
    from oracle import pipelines_ref
    from paper_2512_02371_b200 import pipelines
    g = torch.Generator(device="cpu").manual_seed(sum(shape))
    x = torch.rand(shape, generator=g).bfloat16()
    y = pipelines.resample(x.cuda(), oh, ow, out_dtype=torch.float32)
    torch.cuda.synchronize()
    ref = pipelines_ref.resample(x.float().numpy(), oh, ow)
    assert np.abs(y.cpu().numpy() - ref).max() <= 1e-2
