"""Image-level pipelines restated on the CPU (numpy, f32).

TEST INFRASTRUCTURE ONLY.  Built from the reference's tile semantics: every
1-D pass is the source-form conv statement of make_corpus.conv_update
(tools/make_corpus.py:142-150) evaluated as interp does — f32 products,
taps summed left to right (interp.py:162-167, 203-211), then ``+ acc`` with
acc = 0 (the Store of ``conv``).  tests/golden/ pins that 1-D pass
bit-exactly against interp.run_program on generated tile programs.

What the reference does not define is restated from the paper and chosen
here (parity unpinned, documented in DESIGN.md):
  * Lanczos-3 kernel sinc(x)·sinc(x/3), |x| < 3, output o at
    input coordinate (o + 0.5)·f − 0.5, stretched by max(f, 1), normalised;
  * Gaussian sigma = taps/6 and box 1/taps, centred taps;
  * clamp-to-edge at image borders;
  * separable order: horizontal pass, then vertical (either order is the
    same linear map; only f32 rounding differs);
  * DCT-16 denoise: see dct_denoise.
"""

from __future__ import annotations

import math

import numpy as np


# ------------------------------------------------------------------ weights
def _sinc(x):
    if x == 0.0:
        return 1.0
    return math.sin(math.pi * x) / (math.pi * x)


def lanczos3_weights(n_in, n_out):
    """(first[n_out], weights[n_out, taps]) for Lanczos-3 resampling."""
    f = n_in / n_out
    fs = max(f, 1.0)
    rows = []
    for o in range(n_out):
        c = (o + 0.5) * f - 0.5
        lo = math.ceil(c - 3.0 * fs - 1e-9)
        hi = math.floor(c + 3.0 * fs + 1e-9)
        w = []
        for j in range(lo, hi + 1):
            x = (j - c) / fs
            w.append(_sinc(x) * _sinc(x / 3.0) if abs(x) < 3.0 else 0.0)
        s = sum(w)
        rows.append((lo, [v / s for v in w]))
    taps = max(len(w) for _, w in rows)
    first = np.array([lo for lo, _ in rows], np.int64)
    weights = np.zeros((n_out, taps), np.float32)
    for o, (_, w) in enumerate(rows):
        weights[o, :len(w)] = np.asarray(w, np.float64).astype(np.float32)
    return first, weights


def gaussian_kernel(taps, sigma=None):
    sigma = taps / 6.0 if sigma is None else sigma
    h = (taps - 1) / 2.0
    w = [math.exp(-0.5 * ((t - h) / sigma) ** 2) for t in range(taps)]
    s = sum(w)
    return np.array([v / s for v in w], np.float64).astype(np.float32)


def box_kernel(taps):
    return np.full(taps, 1.0 / taps, np.float32)


def centred_axis(n, kernel):
    kernel = np.asarray(kernel, np.float32)
    taps = len(kernel)
    first = np.arange(n) - (taps - 1) // 2
    return first.astype(np.int64), np.tile(kernel, (n, 1))


# ------------------------------------------------------------------ passes
def axis_pass(x, first, weights, axis):
    """One 1-D pass along `axis`: out[..., o] = (Σ_t x[..., clamp(first[o]+t)]
    · w[o, t]) + 0, f32, t left to right."""
    x = np.moveaxis(np.asarray(x, np.float32), axis, -1)
    n_in = x.shape[-1]
    first = np.asarray(first, np.int64)
    weights = np.asarray(weights, np.float32)
    acc = None
    for t in range(weights.shape[1]):
        idx = np.clip(first + t, 0, n_in - 1)
        term = (x[..., idx] * weights[:, t]).astype(np.float32)
        acc = term if acc is None else (acc + term).astype(np.float32)
    acc = (acc + np.float32(0.0)).astype(np.float32)
    return np.moveaxis(acc, -1, axis)


def separable(img, rows, cols):
    """Horizontal pass then vertical pass; rows/cols = (first, weights)."""
    h = axis_pass(img, cols[0], cols[1], axis=-1)
    return axis_pass(h, rows[0], rows[1], axis=-2)


def resample(img, out_h, out_w):
    img = np.asarray(img, np.float32)
    H, W = img.shape[-2:]
    return separable(img, lanczos3_weights(H, out_h), lanczos3_weights(W, out_w))


def gaussian_blur(img, taps, sigma=None):
    img = np.asarray(img, np.float32)
    k = gaussian_kernel(taps, sigma)
    H, W = img.shape[-2:]
    return separable(img, centred_axis(H, k), centred_axis(W, k))


def box_blur(img, taps):
    img = np.asarray(img, np.float32)
    k = box_kernel(taps)
    H, W = img.shape[-2:]
    return separable(img, centred_axis(H, k), centred_axis(W, k))


# ------------------------------------------------------------------ DCT-16 denoise
def dct_matrix(n=16):
    """Orthonormal DCT-II: D[k][m] = c_k cos(pi (2m + 1) k / 2n)."""
    k = np.arange(n)[:, None]
    m = np.arange(n)[None, :]
    d = np.cos(np.pi * (2 * m + 1) * k / (2 * n)) * np.sqrt(2.0 / n)
    d[0, :] = np.sqrt(1.0 / n)
    return d


def sine_window(n=16):
    """w[m] = sin(pi (m + 0.5) / n): w[m]^2 + w[m + n/2]^2 = 1, so windowed
    analysis + windowed synthesis at stride n/2 reconstructs exactly."""
    return np.sin(np.pi * (np.arange(n) + 0.5) / n)


def dct_window_matrix(n=16):
    """Dw = D·diag(w) in f32 (the analysis / synthesis matrix of a tile)."""
    return (dct_matrix(n) * sine_window(n)[None, :]).astype(np.float32)


def mm_left(A, B):
    """A (n x n) times every tile B (..., n, n) with interp's wmma_mma
    arithmetic (interp.py:459-486): f32 products, k summed left to right
    from k = 0, then C + s with C = 0."""
    A = np.asarray(A, np.float32)
    B = np.asarray(B, np.float32)
    s = (A[:, 0][:, None] * B[..., 0:1, :]).astype(np.float32)
    for k in range(1, A.shape[1]):
        s = (s + A[:, k][:, None] * B[..., k:k + 1, :]).astype(np.float32)
    return (np.float32(0.0) + s).astype(np.float32)


def mm_right(A, B):
    """Every tile A (..., n, n) times B (n x n), wmma_mma arithmetic."""
    A = np.asarray(A, np.float32)
    B = np.asarray(B, np.float32)
    s = (A[..., :, 0:1] * B[0, :]).astype(np.float32)
    for k in range(1, B.shape[0]):
        s = (s + A[..., :, k:k + 1] * B[k, :]).astype(np.float32)
    return (np.float32(0.0) + s).astype(np.float32)


def dct_tiles(img, n=16):
    """(planes, ty, tx, n, n) f32 tiles at stride n/2 over the image extended
    by n/2 on each side with clamp-to-edge; planes flattened."""
    x = np.asarray(img, np.float32)
    h = n // 2
    H, W = x.shape[-2:]
    if H % h or W % h:
        raise ValueError(f"image {H}x{W} must be a multiple of {h}")
    x = x.reshape((-1, H, W))
    xp = np.pad(x, ((0, 0), (h, h), (h, h)), mode="edge")
    ty, tx = H // h + 1, W // h + 1
    s = xp.strides
    return np.lib.stride_tricks.as_strided(
        xp, shape=(x.shape[0], ty, tx, n, n), strides=(s[0], s[1] * h, s[2] * h, s[1], s[2])).copy()


def dct_coefficients(img, n=16):
    """Forward transform of every tile: C = (Dw · T) · Dwᵀ, two wmma_mma
    products per tile (pinned bitwise to reference-run programs,
    tests/golden dct_*)."""
    Dw = dct_window_matrix(n)
    return mm_right(mm_left(Dw, dct_tiles(img, n)), np.ascontiguousarray(Dw.T))


def dct_core(C, threshold, mode):
    """Coring of every non-DC coefficient (hard: |c| < threshold -> 0; soft:
    shrink towards 0 by threshold); f32."""
    C = np.asarray(C, np.float32)
    dc = C[..., 0, 0].copy()
    if mode == "hard":
        C = np.where(np.abs(C) < threshold, np.float32(0), C).astype(np.float32)
    elif mode == "soft":
        C = (np.sign(C) * np.maximum(np.abs(C) - np.float32(threshold), np.float32(0))).astype(np.float32)
    else:
        raise ValueError(mode)
    C[..., 0, 0] = dc
    return C


def dct_overlap_add(R, H, W, n=16):
    """Overlap-add of the inverse tiles R (planes, ty, tx, n, n): each output
    pixel is the f32 sum of its four tiles in phase order (0,0), (0,1),
    (1,0), (1,1), starting from 0; returns (planes, H, W)."""
    h = n // 2
    P = R.shape[0]
    out = np.zeros((P, H + 2 * h, W + 2 * h), np.float32)
    for py in range(2):
        for px in range(2):
            sub = R[:, py::2, px::2]
            ny, nx = sub.shape[1], sub.shape[2]
            blk = sub.transpose(0, 1, 3, 2, 4).reshape(P, ny * n, nx * n)
            out[:, py * h:py * h + ny * n, px * h:px * h + nx * n] += blk
    return out[:, h:h + H, h:h + W]


def dct_denoise(img, threshold, mode="hard", n=16):
    """Transform-domain coring, restated.

    Tiles of n x n at stride n/2 over the image extended by n/2 on each side
    (clamp-to-edge); each tile is windowed (sine window, separable), DCT-II'd
    (C = Dw T Dwᵀ with Dw = D·diag(w)), cored (hard: |c| < threshold -> 0;
    soft: shrink towards 0 by threshold; the DC bin is always kept), inverse
    transformed with the same window (Dwᵀ C Dw) and overlap-added.  With
    threshold 0 the output equals the input (up to f32 rounding).
    Image height/width must be multiples of n/2.

    The four 16x16x16 products per tile are interp's wmma_mma (f32 products,
    left-to-right k, + 0): pinned bitwise to programs run by the reference
    (oracle/make_golden.py, tests/golden dct_*); tiling, coring and the
    overlap-add order are this restatement's choices (the reference has no
    code for them)."""
    x = np.asarray(img, np.float32)
    H, W = x.shape[-2:]
    lead = x.shape[:-2]
    Dw = dct_window_matrix(n)
    C = dct_core(dct_coefficients(x, n), threshold, mode)
    R = mm_right(mm_left(np.ascontiguousarray(Dw.T), C), Dw)
    return dct_overlap_add(R, H, W, n).reshape(lead + (H, W)).astype(np.float32)


def dct_flip_mask(img, threshold, eps, n=16):
    """Pixels whose hard-coring result depends on a coefficient within `eps`
    of the threshold: any non-DC coefficient of any tile covering the pixel
    with ||c| - threshold| <= eps.  An implementation whose forward
    coefficients are within eps of these can decide such a coefficient
    either way; every other pixel has an unambiguous result."""
    x = np.asarray(img, np.float32)
    H, W = x.shape[-2:]
    C = dct_coefficients(x, n)
    near = np.abs(np.abs(C) - np.float32(threshold)) <= eps
    near[..., 0, 0] = False
    tile = near.any(axis=(-1, -2))  # (P, ty, tx)
    h = n // 2
    P, ty, tx = tile.shape
    m = np.zeros((P, H + 2 * h, W + 2 * h), bool)
    for p, i, j in zip(*np.nonzero(tile)):
        m[p, h * i:h * i + n, h * j:h * j + n] = True
    return m[:, h:h + H, h:h + W].reshape(x.shape[:-2] + (H, W))
