"""Out-of-bounds write checks for every kernel family (the pool does not
allow compute-sanitizer: runs under it have left GPUs needing a reset).

Each kernel writes its output through the C ABI into a view of a larger
buffer: canary bands before and after the output, and padding columns
between rows (row stride > width).  The canaries must survive bit for bit,
and the strided output must equal a compact call of the same pipeline.
The ABI's row contract (include/tensorsel_b200.h): a row is written in
whole 16-byte units — TMA stores fill the last partial 16 bytes of a row —
so the bytes up to the next 16-byte boundary belong to the row (row strides
are multiples of 16 bytes); everything past that must stay untouched.
Inputs sit between NaN guard bands; a read outside the image would turn
outputs into NaN.  Ragged sizes exercise the edge tiles of every kernel.
"""

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

CANARY = 0x7F7F  # a bf16 / f16 bit pattern no kernel produces from finite inputs


def _torch():
    import torch
    return torch


def _guarded_input(x, pad_cols=8, guard=4096):
    """x (P, H, W) bf16/f32 -> (view with row stride W + pad_cols inside a
    NaN-guarded buffer, row stride)."""
    torch = _torch()
    P, H, W = x.shape
    rs = -(-W // 8) * 8 + pad_cols  # 16-byte rows (TMA)
    buf = torch.full((2 * guard + P * H * rs,), float("nan"), dtype=x.dtype, device=x.device)
    v = buf[guard:guard + P * H * rs].view(P, H, rs)
    v[:, :, :W] = x
    return v, rs, buf


def _guarded_output(P, H, W, dtype, pad_cols=8, guard=4096):
    torch = _torch()
    rs = -(-W // 8) * 8 + pad_cols  # 16-byte rows (TMA)
    n = 2 * guard + P * H * rs
    if dtype == torch.float32:
        buf = torch.empty((n,), dtype=torch.int32, device="cuda").fill_(0x7F7F7F7F).view(torch.float32)
    else:
        buf = torch.empty((n,), dtype=torch.int16, device="cuda").fill_(CANARY).view(dtype)
    out = buf[guard:guard + P * H * rs].view(P, H, rs)
    return out, rs, buf


def _canaries_intact(buf, out, W):
    torch = _torch()
    bits = buf.view(torch.int32 if buf.dtype == torch.float32 else torch.int16)
    want = 0x7F7F7F7F if buf.dtype == torch.float32 else CANARY
    inner = torch.zeros_like(bits, dtype=torch.bool)
    o0 = out.data_ptr() - buf.data_ptr()
    o0 //= buf.element_size()
    P, H, rs = out.shape
    W16 = -(-W * buf.element_size() // 16) * 16 // buf.element_size()  # the row's 16-byte units
    idx = torch.arange(P * H * rs, device=buf.device).view(P, H, rs)[:, :, :W16].reshape(-1) + o0
    inner[idx] = True
    return bool(((bits == want) | inner).all())


@pytest.mark.parametrize("shape,oh,ow,out_dtype", [
    ((3, 270, 484), 135, 242, "bf16"),
    ((2, 133, 200), 66, 100, "f32"),
    ((1, 1000, 1504), 400, 600, "bf16"),   # non-integer factor, fused
    ((1, 900, 904), 60, 64, "f32"),        # 15x: the two axis passes
])
def test_resample_writes_only_its_output(shape, oh, ow, out_dtype):
    torch = _torch()
    from paper_2512_02371_b200 import _lib, axis, pipelines
    dt = torch.bfloat16 if out_dtype == "bf16" else torch.float32
    g = torch.Generator(device="cpu").manual_seed(sum(shape))
    x = torch.rand(shape, generator=g).bfloat16().cuda()
    want = pipelines.resample(x, oh, ow, out_dtype=dt)
    P, H, W = shape
    xin, irs, _ = _guarded_input(x)
    out, ors, buf = _guarded_output(P, oh, ow, dt)
    ra, ca = axis.lanczos3(H, oh, 0), axis.lanczos3(W, ow, 0)
    ts_out = _lib.TS_BF16 if dt == torch.bfloat16 else _lib.TS_F32
    lib = _lib.load()
    s = torch.cuda.current_stream().cuda_stream
    if pipelines.fused_supported(ra, ca, P, ts_out):
        _lib.check(lib.ts_separable_run(ra.handle, ca.handle, P, xin.data_ptr(), irs, irs * H,
                                        _lib.TS_BF16, out.data_ptr(), ors, ors * oh, ts_out, s))
    else:
        mid, mrs, mbuf = _guarded_output(P, oh, W, torch.bfloat16)
        _lib.check(lib.ts_axis_pass(ra.handle, 0, P, H, W, xin.data_ptr(), irs, irs * H,
                                    mid.data_ptr(), mrs, mrs * oh, _lib.TS_BF16, s))
        _lib.check(lib.ts_axis_pass(ca.handle, 1, P, oh, W, mid.data_ptr(), mrs, mrs * oh,
                                    out.data_ptr(), ors, ors * oh, ts_out, s))
        torch.cuda.synchronize()
        assert _canaries_intact(mbuf, mid, W)
    torch.cuda.synchronize()
    assert _canaries_intact(buf, out, ow)
    assert torch.equal(out[:, :, :ow].contiguous().view(torch.int16 if dt == torch.bfloat16
                                                        else torch.int32),
                       want.view(torch.int16 if dt == torch.bfloat16 else torch.int32))


@pytest.mark.parametrize("shape,soft,out_dtype", [
    ((2, 136, 248), 0, "bf16"), ((1, 96, 520), 1, "f32"), ((3, 120, 128), 0, "f32"),
])
def test_dct16_writes_only_its_output(shape, soft, out_dtype):
    torch = _torch()
    from paper_2512_02371_b200 import _lib, pipelines
    dt = torch.bfloat16 if out_dtype == "bf16" else torch.float32
    g = torch.Generator(device="cpu").manual_seed(7)
    x = torch.rand(shape, generator=g).bfloat16().cuda()
    want = pipelines.denoise_dct16(x, 0.15, "soft" if soft else "hard", out_dtype=dt)
    P, H, W = shape
    xin, irs, _ = _guarded_input(x)
    out, ors, buf = _guarded_output(P, H, W, dt)
    _lib.check(_lib.load().ts_denoise_dct16(
        xin.data_ptr(), irs, irs * H, _lib.TS_BF16, out.data_ptr(), ors, ors * H,
        _lib.TS_BF16 if dt == torch.bfloat16 else _lib.TS_F32, P, H, W, 0.15, soft,
        torch.cuda.current_stream().cuda_stream))
    torch.cuda.synchronize()
    assert _canaries_intact(buf, out, W)
    iv = torch.int16 if dt == torch.bfloat16 else torch.int32
    assert torch.equal(out[:, :, :W].contiguous().view(iv), want.view(iv))


@pytest.mark.parametrize("shape,taps", [((3, 270, 484), 12), ((2, 97, 132), 9), ((1, 64, 68), 31)])
def test_f32_kernel_writes_only_its_output(shape, taps):
    torch = _torch()
    from paper_2512_02371_b200 import _lib, axis, filters, pipelines
    g = torch.Generator(device="cpu").manual_seed(3)
    x = torch.rand(shape, generator=g).cuda()
    P, H, W = shape
    if taps == 12:
        oh, ow = H // 2, W // 2
        ra, ca = axis.lanczos3(H, oh, 0), axis.lanczos3(W, ow, 0)
        want = pipelines.resample(x, oh, ow, out_dtype=torch.float32)
    else:
        oh, ow = H, W
        k = filters.gaussian_taps(taps)
        ra, ca = axis.convolution(H, k, 0), axis.convolution(W, k, 0)
        want = pipelines.gaussian_blur(x, taps, out_dtype=torch.float32)
    ur, uc = ra.uniform, ca.uniform
    xin, irs, _ = _guarded_input(x)
    out, ors, buf = _guarded_output(P, oh, ow, torch.float32)
    wr, wc = ra.device_weights(), ca.device_weights()
    _lib.check(_lib.load().ts_separable_f32_ep(
        P, xin.data_ptr(), H, W, irs, irs * H, ur[0], ur[1], ur[2], wr.data_ptr(), oh, uc[2],
        wc.data_ptr(), ow, out.data_ptr(), ors, ors * oh, _lib.TS_F32, 0, None,
        torch.cuda.current_stream().cuda_stream))
    torch.cuda.synchronize()
    assert _canaries_intact(buf, out, ow)
    assert torch.equal(out[:, :, :ow].contiguous().view(torch.int32), want.view(torch.int32))
