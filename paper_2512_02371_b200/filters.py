"""Resampling / filter tap generators (host side, run once per axis).

The reference ships only the Toeplitz-family matrix *shapes*
(layout.py:1-135); the kernels' *values* come from the paper:

* Lanczos-3 pre-filter ``sinc(x)·sinc(x/3)`` for ``|x| < 3``, applied
  separably, stretched by the scale factor when downsampling
  (§V-C "Resampling by a non-integer factor").
* Gaussian (sigma = taps/6) and box (1/taps) separable filters for the
  convolution case study.

Every generator returns ``(first, weights)``: output ``o`` reads inputs
``first[o] + t`` (t < taps, unclamped) with ``weights[o, t]``.  The axis
builder folds out-of-range indices onto the edge sample (clamp-to-edge).
These definitions are restated independently in ``oracle/pipelines_ref.py``.
"""

from __future__ import annotations


import numpy as np


def lanczos3(x):
    """L(x) = sinc(x)·sinc(x/3) on |x| < 3, 0 elsewhere."""
    x = np.asarray(x, dtype=np.float64)
    out = np.sinc(x) * np.sinc(x / 3.0)
    return np.where(np.abs(x) < 3.0, out, 0.0)


def lanczos3_axis(n_in: int, n_out: int):
    """Lanczos-3 resampling of an axis of n_in samples to n_out samples.

    Output sample ``o`` sits at input coordinate ``c = (o + 0.5)·f − 0.5``
    with ``f = n_in / n_out``; the filter is stretched by ``max(f, 1)`` so it
    rejects frequencies above the output Nyquist rate when downsampling.
    Taps cover ``[c − 3·fs, c + 3·fs]`` and are normalised to sum 1.  For an
    integer factor ``s`` this is the strided Toeplitz matrix of
    ``layout.strided_toeplitz`` (layout.py:92-94) with ``l = 6s`` taps; for
    s = 2 the first tap is at ``2o − 5``.
    """
    if n_in < 1 or n_out < 1:
        raise ValueError("axis lengths must be >= 1")
    f = n_in / n_out
    fs = max(f, 1.0)
    o = np.arange(n_out, dtype=np.float64)
    c = (o + 0.5) * f - 0.5
    lo = np.ceil(c - 3.0 * fs - 1e-9).astype(np.int64)
    hi = np.floor(c + 3.0 * fs + 1e-9).astype(np.int64)
    taps = int((hi - lo).max()) + 1
    t = np.arange(taps)
    idx = lo[:, None] + t[None, :]
    w = lanczos3((idx - c[:, None]) / fs)
    w = np.where(idx <= hi[:, None], w, 0.0)
    w /= w.sum(axis=1, keepdims=True)
    return lo.astype(np.int32), w.astype(np.float32)


def gaussian_taps(taps: int, sigma: float | None = None):
    """Normalised Gaussian, sigma = taps/6 by default."""
    if taps < 1:
        raise ValueError("taps must be >= 1")
    sigma = taps / 6.0 if sigma is None else float(sigma)
    h = (taps - 1) / 2.0
    x = np.arange(taps, dtype=np.float64) - h
    w = np.exp(-0.5 * (x / sigma) ** 2)
    return (w / w.sum()).astype(np.float32)


def box_taps(taps: int):
    if taps < 1:
        raise ValueError("taps must be >= 1")
    return np.full(taps, 1.0 / taps, dtype=np.float32)


def conv_axis(n: int, kernel):
    """Same-size 'centred' convolution of an axis: output o reads
    inputs o − (taps−1)//2 + t.  This is the plain Toeplitz matrix
    (layout.toeplitz_matrix, layout.py:87-89) shifted to centre the kernel."""
    kernel = np.asarray(kernel, dtype=np.float32)
    taps = len(kernel)
    first = (np.arange(n) - (taps - 1) // 2).astype(np.int32)
    w = np.broadcast_to(kernel, (n, taps)).copy()
    return first, w


def downsample_offset(l: int, s: int) -> int:
    """Offset of the first tap for an even-length symmetric l-tap kernel at
    stride s, centred on output pixel o (centre s·o + (s−1)/2)."""
    return -((l - s) // 2)


def ceil_div(a: int, b: int) -> int:
    return -(-a // b)


__all__ = ["lanczos3", "lanczos3_axis", "gaussian_taps", "box_taps", "conv_axis",
           "downsample_offset", "ceil_div"]
