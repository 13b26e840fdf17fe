"""Image pipelines that are linear transforms in disguise, on B200.

The paper's case studies (§V) as one call each, executed by the
fused sm_100a kernels behind the C ABI:

* :func:`resample` — separable Lanczos-3 resampling (integer or non-integer
  factor).  ``downsample2x`` is the 2x case of configs 1,
  2 and 5.
* :func:`filter_separable`, :func:`gaussian_blur`, :func:`box_blur` —
  same-size separable convolution (config 3).

Images are planar: a tensor ``(..., H, W)`` is a stack of planes (RGB
counts as 3 planes).  bf16 inputs run on the tensor cores (f32 accumulate);
f32 inputs on uniform axes (exact-2x Lanczos-3, centred filters) run in f32
on the FMA pipe (``ts_separable_f32_ep``; bit-identical to the reference
with ``F32_EXACT``), other f32 inputs are cast to bf16 on the device.  Edges are clamp-to-edge.  There is
no CPU path: without the native library or a CUDA device these raise.

Every pipeline takes an optional output epilogue, applied inside the
producing kernel to the f32 result before the final cast (the "clamp /
normalise" step): ``y = clamp(x * scale + bias, *clamp)``, e.g.
``resample(x, 1080, 1920, clamp=(0, 1))`` removes Lanczos overshoot and
``scale=255.0`` rescales to 8-bit range.  Without these arguments the
kernels without an epilogue run.
"""

from __future__ import annotations

import math
import os

import numpy as np

from . import _lib, axis as _axis, filters
from .errors import NoDevice


def _torch():
    import torch
    return torch


def _check_device(x):
    torch = _torch()
    if not isinstance(x, torch.Tensor) or not x.is_cuda:
        raise NoDevice("pipelines operate on CUDA tensors; move the image to the GPU first")
    return x.device.index if x.device.index is not None else torch.cuda.current_device()


def _as_planes_bf16(x, stream):
    """View/copy x (..., H, W) as a (P, H, Wp) bf16 buffer with Wp % 8 == 0."""
    torch = _torch()
    H, W = x.shape[-2], x.shape[-1]
    P = math.prod(x.shape[:-2]) if x.dim() > 2 else 1
    if x.dtype == torch.bfloat16 and W % 8 == 0 and x.is_contiguous():
        return x.reshape(P, H, W), W
    Wp = -(-W // 8) * 8
    if x.dtype == torch.float32 and x.is_contiguous() and W == Wp:
        buf = torch.empty((P, H, W), dtype=torch.bfloat16, device=x.device)
        _lib.check(_lib.load().ts_cast_f32_bf16(x.data_ptr(), buf.data_ptr(), x.numel(), stream),
                   "ts_cast_f32_bf16")
        return buf, W
    if x.dtype not in (torch.bfloat16, torch.float32):
        raise TypeError(f"unsupported input dtype {x.dtype} (bf16 or f32)")
    buf = torch.zeros((P, H, Wp), dtype=torch.bfloat16, device=x.device)
    buf[:, :, :W].copy_(x.reshape(P, H, W))
    return buf, Wp


_FUSED = {}


def fused_supported(ra, ca, planes=1, ts_out=None) -> bool:
    """Whether the fused separable kernel tiles these axes (otherwise the
    pipelines run two ``ts_axis_pass`` launches).  Memoised per axis pair."""
    key = (ra, ca, planes, ts_out or _lib.TS_BF16)
    ok = _FUSED.get(key)
    if ok is not None:
        return ok
    import ctypes
    lib = _lib.load()
    out8 = (ctypes.c_int * 8)()
    st = lib.ts_separable_plan(ra.handle, ca.handle, planes, key[3], out8)
    if st not in (0, 6):  # 6 = TS_ERR_UNSUPPORTED: geometry
        _lib.check(st, "ts_separable_plan")
    _FUSED[key] = ok = st == 0
    return ok


def _stream(x):
    """Raw cudaStream_t of the current stream on x's device."""
    torch = _torch()
    get = getattr(torch._C, "_cuda_getCurrentRawStream", None)
    if get is not None:
        return get(x.device.index if x.device.index is not None else torch.cuda.current_device())
    return torch.cuda.current_stream(x.device).cuda_stream


def _epilogue(clamp, scale, bias):
    """ts_epilogue for the keyword arguments, or None (no epilogue)."""
    if clamp is None and scale is None and bias is None:
        return None
    lo, hi = (-math.inf, math.inf) if clamp is None else (float(clamp[0]), float(clamp[1]))
    if lo > hi:
        raise ValueError(f"clamp=({lo}, {hi}): lower bound above upper bound")
    return _lib.Epilogue(1.0 if scale is None else float(scale),
                         0.0 if bias is None else float(bias), lo, hi)


def _ep_ptr(ep):
    import ctypes
    return ctypes.byref(ep)


# (stride, taps, base & 3) csrc/separable_f32.cu instantiates
_F32_KERNELS = frozenset({(2, 12, 3), (1, 9, 0), (1, 15, 1), (1, 21, 2), (1, 31, 1)})

# f32 images: True = the reference's separate product / sum roundings
# (bit-identical f32 output, slower), False = one fused multiply-add per tap.
# Default from TSB_F32_EXACT=1 in the environment.
F32_EXACT = os.environ.get("TSB_F32_EXACT", "0") == "1"


def _run_f32(x, ra, ca, out_dtype, ep, stream):
    """f32 images through ``ts_separable_f32_ep`` (FMA pipe, the f32 image
    read once; bit-identical to the reference's f32 evaluation when
    ``F32_EXACT``) when
    both axes are uniform-stride with an instantiated (stride, taps);
    otherwise None and the caller takes the bf16 tensor-core path."""
    ur, uc = ra.uniform, ca.uniform
    if (ur is None or uc is None or ur[:2] != uc[:2]
            or (uc[0], uc[1], uc[2] & 3) not in _F32_KERNELS):
        return None
    torch = _torch()
    H, W = x.shape[-2], x.shape[-1]
    P = math.prod(x.shape[:-2]) if x.dim() > 2 else 1
    lead = x.shape[:-2]
    rs = W
    if W % 4 or x.data_ptr() % 16:
        # the window is one TMA box: rows must start on 16 bytes -> a pitched copy
        rs = -(-W // 4) * 4
        xp = torch.empty((P, H, rs), dtype=torch.float32, device=x.device)
        xp[:, :, :W] = x.reshape(P, H, W)
        x = xp
    oh, ow = ra.n_out, ca.n_out
    out = torch.empty((P, oh, ow), dtype=out_dtype, device=x.device)
    ts_out = _lib.TS_BF16 if out_dtype == torch.bfloat16 else _lib.TS_F32
    wr, wc = ra.device_weights(), ca.device_weights()
    _lib.check(_lib.load().ts_separable_f32_ep(
        P, x.data_ptr(), H, W, rs, rs * H, ur[0], ur[1], ur[2], wr.data_ptr(), oh, uc[2],
        wc.data_ptr(), ow, out.data_ptr(), ow, ow * oh, ts_out, 1 if F32_EXACT else 0,
        None if ep is None else _ep_ptr(ep), stream), "ts_separable_f32_ep")
    return out.reshape(*lead, oh, ow)


def _run(x, ra, ca, out_dtype, ep=None):
    torch = _torch()
    _check_device(x)
    stream = _stream(x)
    H, W = x.shape[-2], x.shape[-1]
    if ra.n_in != H or ca.n_in != W:
        raise ValueError(f"axes expect {ra.n_in} x {ca.n_in}, image is {H} x {W}")
    out_dtype = out_dtype or (x.dtype if x.dtype in (torch.bfloat16, torch.float32)
                              else torch.bfloat16)
    if out_dtype not in (torch.bfloat16, torch.float32):
        raise TypeError(f"unsupported out_dtype {out_dtype} (bf16 or f32)")
    oh, ow = ra.n_out, ca.n_out
    if x.numel() == 0:  # empty batch: nothing to launch
        return torch.empty((*x.shape[:-2], oh, ow), dtype=out_dtype, device=x.device)
    if x.dtype == torch.float32 and x.is_contiguous():
        y = _run_f32(x, ra, ca, out_dtype, ep, stream)
        if y is not None:
            return y
    inb, in_rs = _as_planes_bf16(x, stream)
    P = inb.shape[0]
    align = 8 if out_dtype == torch.bfloat16 else 4
    owp = -(-ow // align) * align
    out = torch.empty((P, oh, owp), dtype=out_dtype, device=x.device)
    ts_out = _lib.TS_BF16 if out_dtype == torch.bfloat16 else _lib.TS_F32
    lib = _lib.load()
    if fused_supported(ra, ca, P, ts_out):
        if ep is None:
            _lib.check(lib.ts_separable_run(
                ra.handle, ca.handle, P, inb.data_ptr(), in_rs, in_rs * H, _lib.TS_BF16,
                out.data_ptr(), owp, owp * oh, ts_out, stream), "ts_separable_run")
        else:
            _lib.check(lib.ts_separable_run_ep(
                ra.handle, ca.handle, P, inb.data_ptr(), in_rs, in_rs * H, _lib.TS_BF16,
                out.data_ptr(), owp, owp * oh, ts_out, _ep_ptr(ep), stream), "ts_separable_run_ep")
    else:
        # windows too wide for the fused tile (large downscale factors, very
        # wide filters): two axis passes, bf16 intermediate in HBM — the same
        # rounding point as the fused kernel's intermediate
        mid = torch.empty((P, oh, in_rs), dtype=torch.bfloat16, device=x.device)
        _lib.check(lib.ts_axis_pass(ra.handle, 0, P, H, W, inb.data_ptr(), in_rs, in_rs * H,
                                    mid.data_ptr(), in_rs, in_rs * oh, _lib.TS_BF16, stream),
                   "ts_axis_pass")
        if ep is None:
            _lib.check(lib.ts_axis_pass(ca.handle, 1, P, oh, W, mid.data_ptr(), in_rs, in_rs * oh,
                                        out.data_ptr(), owp, owp * oh, ts_out, stream),
                       "ts_axis_pass")
        else:  # the epilogue belongs to the last pass
            _lib.check(lib.ts_axis_pass_ep(ca.handle, 1, P, oh, W, mid.data_ptr(), in_rs,
                                           in_rs * oh, out.data_ptr(), owp, owp * oh, ts_out,
                                           _ep_ptr(ep), stream), "ts_axis_pass_ep")
    if owp != ow:
        out = out[:, :, :ow]
    return out.reshape(*x.shape[:-2], oh, ow)


def resample(x, out_h: int, out_w: int, *, out_dtype=None, clamp=None, scale=None, bias=None):
    """Separable Lanczos-3 resample of planar images to (out_h, out_w)."""
    dev = _check_device(x)
    H, W = x.shape[-2], x.shape[-1]
    ra = _axis.lanczos3(H, out_h, dev)
    ca = _axis.lanczos3(W, out_w, dev)
    return _run(x, ra, ca, out_dtype, _epilogue(clamp, scale, bias))


def downsample2x(x, *, out_dtype=None, clamp=None, scale=None, bias=None):
    """Lanczos-3 2x downsample (configs 1/2: 1080p->540p, 4K->1080p)."""
    H, W = x.shape[-2], x.shape[-1]
    return resample(x, H // 2, W // 2, out_dtype=out_dtype, clamp=clamp, scale=scale, bias=bias)


def upsample2x(x, *, out_dtype=None, clamp=None, scale=None, bias=None):
    """Lanczos-3 2x upsample: the polyphase Toeplitz case (layout.polyphase_toeplitz,
    layout.py:97-103) — each output phase is a 6-tap filter."""
    H, W = x.shape[-2], x.shape[-1]
    return resample(x, 2 * H, 2 * W, out_dtype=out_dtype, clamp=clamp, scale=scale, bias=bias)


def filter_separable(x, kernel_v, kernel_h=None, *, out_dtype=None, clamp=None, scale=None,
                     bias=None):
    """Same-size separable convolution (centred taps, clamp-to-edge)."""
    dev = _check_device(x)
    kernel_h = kernel_v if kernel_h is None else kernel_h
    H, W = x.shape[-2], x.shape[-1]
    ra = _axis.convolution(H, kernel_v, dev)
    ca = _axis.convolution(W, kernel_h, dev)
    return _run(x, ra, ca, out_dtype, _epilogue(clamp, scale, bias))


def gaussian_blur(x, taps: int, sigma: float | None = None, *, out_dtype=None, clamp=None,
                  scale=None, bias=None):
    k = filters.gaussian_taps(taps, sigma)
    return filter_separable(x, k, k, out_dtype=out_dtype, clamp=clamp, scale=scale, bias=bias)


def box_blur(x, taps: int, *, out_dtype=None, clamp=None, scale=None, bias=None):
    k = filters.box_taps(taps)
    return filter_separable(x, k, k, out_dtype=out_dtype, clamp=clamp, scale=scale, bias=bias)


def resample_filter(x, out_h: int, out_w: int, taps: int = 9, sigma: float | None = None, *,
                    out_dtype=None, clamp=None, scale=None, bias=None):
    """Lanczos-3 resample to (out_h, out_w), then a `taps`-tap Gaussian at the
    output resolution (config 5) — fused into ONE separable pass by composing
    the two banded axes on the host (no intermediate image in HBM)."""
    dev = _check_device(x)
    H, W = x.shape[-2], x.shape[-1]
    k = filters.gaussian_taps(taps, sigma)
    ra = _axis.resample_filter(H, out_h, k, dev)
    ca = _axis.resample_filter(W, out_w, k, dev)
    return _run(x, ra, ca, out_dtype, _epilogue(clamp, scale, bias))


def denoise_dct16(x, threshold: float = 0.15, mode: str = "hard", *, out_dtype=None,
                  clamp=None, scale=None, bias=None):
    """DCT-16 transform-domain coring (config 4): 16x16
    tiles at stride 8, sine-windowed DCT-II, coefficients below `threshold`
    zeroed (mode="hard", the paper's coring) or shrunk (mode="soft"), DC
    kept, windowed inverse + overlap-add, clamp-to-edge.  One fused kernel.
    Height and width must be multiples of 8."""
    torch = _torch()
    _check_device(x)
    if mode not in ("hard", "soft"):
        raise ValueError("mode must be 'hard' or 'soft'")
    stream = _stream(x)
    H, W = x.shape[-2], x.shape[-1]
    out_dtype = out_dtype or (x.dtype if x.dtype in (torch.bfloat16, torch.float32)
                              else torch.bfloat16)
    if out_dtype not in (torch.bfloat16, torch.float32):
        raise TypeError(f"unsupported out_dtype {out_dtype} (bf16 or f32)")
    if x.numel() == 0:
        return torch.empty(x.shape, dtype=out_dtype, device=x.device)
    inb, in_rs = _as_planes_bf16(x, stream)
    P = inb.shape[0]
    align = 8 if out_dtype == torch.bfloat16 else 4
    owp = -(-W // align) * align
    out = torch.empty((P, H, owp), dtype=out_dtype, device=x.device)
    ep = _epilogue(clamp, scale, bias)
    args = (inb.data_ptr(), in_rs, in_rs * H, _lib.TS_BF16, out.data_ptr(), owp, owp * H,
            _lib.TS_BF16 if out_dtype == torch.bfloat16 else _lib.TS_F32, P, H, W,
            float(threshold), 1 if mode == "soft" else 0)
    if ep is None:
        _lib.check(_lib.load().ts_denoise_dct16(*args, stream), "ts_denoise_dct16")
    else:
        _lib.check(_lib.load().ts_denoise_dct16_ep(*args, _ep_ptr(ep), stream),
                   "ts_denoise_dct16_ep")
    if owp != W:
        out = out[:, :, :W]
    return out.reshape(*x.shape[:-2], H, W)


def separable(x, rows: "_axis.Axis", cols: "_axis.Axis", *, out_dtype=None, clamp=None,
              scale=None, bias=None):
    """Apply explicit axes: out = rows · x · colsᵀ per plane."""
    return _run(x, rows, cols, out_dtype, _epilogue(clamp, scale, bias))


_LANES = {}


def run_from_host(fn, host_in, host_out, *, chunk_planes: int = 3, lanes: int = 3):
    """Stream a batch of planes from (pinned) host memory through `fn` (any
    pipeline of this module) and back: chunks of `chunk_planes` planes rotate
    over `lanes` CUDA streams, so the host->device copy of one chunk, the
    kernels of another and the device->host copy of a third overlap (PCIe is
    full duplex).  Enqueued on the current device; the current stream waits
    for all of it, so synchronising that stream (or the device) completes the
    batch.  host_out must be preallocated with fn's output shape."""
    torch = _torch()
    dev = torch.device("cuda", torch.cuda.current_device())
    cur = torch.cuda.current_stream(dev)
    key = (dev.index, lanes)
    streams = _LANES.get(key)
    if streams is None:
        streams = _LANES[key] = [torch.cuda.Stream(dev) for _ in range(lanes)]
    start = torch.cuda.Event()
    start.record(cur)
    P = host_in.shape[0]
    for i, c0 in enumerate(range(0, P, chunk_planes)):
        n = min(chunk_planes, P - c0)
        s = streams[i % lanes]
        s.wait_event(start)
        with torch.cuda.stream(s):
            xd = host_in[c0:c0 + n].to(dev, non_blocking=True)
            y = fn(xd)
            host_out[c0:c0 + n].copy_(y, non_blocking=True)
            xd.record_stream(s)
            y.record_stream(s)
    for s in streams:
        cur.wait_stream(s)
    return host_out
