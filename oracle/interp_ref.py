"""Restated interpreter semantics for the conv-family hot path.

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).  Each function cites the
reference lines it restates; values are carried in float32 exactly like the
reference (bf16/f16 in an f32 carrier).
"""

from __future__ import annotations

import numpy as np


# --------------------------------------------------------------- rounding
def round_bf16(x):
    """interp.round_bf16 (interp.py:62-69): RNE into bf16, f32 carrier."""
    a = np.asarray(x, dtype=np.float32)
    u = a.view(np.uint32).astype(np.uint64)
    r = ((u + 0x7FFF + ((u >> 16) & 1)) >> 16) << 16
    out = r.astype(np.uint32).view(np.float32)
    return np.where(np.isnan(a), np.float32(np.nan), out).astype(np.float32)


def round_f16(x):
    """interp.round_f16 (interp.py:72-77)."""
    a = np.asarray(x, dtype=np.float32)
    with np.errstate(over="ignore"):
        return a.astype(np.float16).astype(np.float32)


def round_to_kind(x, kind):
    """interp.round_to_kind (interp.py:80-87)."""
    if kind == "bf16":
        return round_bf16(x)
    if kind == "f16":
        return round_f16(x)
    return np.asarray(x, dtype=np.float32)


# --------------------------------------------------------------- generator
class SplitMix64:
    """interp.SplitMix64 (interp.py:94-115)."""

    M = (1 << 64) - 1

    def __init__(self, seed):
        self.s = seed & self.M

    def next_u64(self):
        self.s = (self.s + 0x9E3779B97F4A7C15) & self.M
        z = self.s
        z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & self.M
        z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & self.M
        return z ^ (z >> 31)

    def uniform(self):
        return (self.next_u64() >> 11) / float(1 << 53) * 2.0 - 1.0

    def small_int(self):
        return self.next_u64() >> 60


def random_fill(params, seed):
    """interp.random_inputs (interp.py:622-634) for a list of
    (name, kind, length); one stream, declaration order."""
    rng = SplitMix64(seed)
    out = {}
    for name, kind, length in params:
        if kind == "i32":
            out[name] = np.array([rng.small_int() for _ in range(length)], np.int64)
        else:
            raw = np.array([rng.uniform() for _ in range(length)], np.float32)
            out[name] = round_to_kind(raw, kind)
    return out


# --------------------------------------------------------------- reductions
def foldl_rows(terms):
    """Left-to-right f32 sum along the last axis (interp._foldl, interp.py:162-167)."""
    terms = np.asarray(terms, dtype=np.float32)
    acc = terms[..., 0].copy()
    for j in range(1, terms.shape[-1]):
        acc = (acc + terms[..., j]).astype(np.float32)
    return acc


def conv_statement(I, K, base_i, taps, stride, n_out, acc=None):
    """Source-form conv update (make_corpus.conv_update, tools/make_corpus.py:142-150):
    out[x] = VectorReduceAdd(I[base + stride*x + t] * K[t]) + acc[x], the
    reduction left to right over t (interp.py:203-211), products in f32."""
    I = np.asarray(I, np.float32)
    K = np.asarray(K, np.float32)
    idx = base_i + stride * np.arange(n_out)[:, None] + np.arange(taps)[None, :]
    prods = (I[idx] * K[None, :taps]).astype(np.float32)
    s = foldl_rows(prods)
    acc = np.zeros(n_out, np.float32) if acc is None else np.asarray(acc, np.float32)
    return (s + acc).astype(np.float32)


def wmma_mma(a, b, c, m, k, n):
    """interp eval_intrinsic 'wmma_mma' (interp.py:459-486): products in
    f32, k summed left to right from k=0, then + C."""
    am = np.asarray(a, np.float32).reshape(m, k)
    bm = np.asarray(b, np.float32).reshape(k, n)
    prods = am[:, :, None] * bm[None, :, :]
    s = prods[:, 0, :].copy()
    for kk in range(1, k):
        s = (s + prods[:, kk, :]).astype(np.float32)
    return (np.asarray(c, np.float32).reshape(m, n) + s).reshape(-1)


def tile_gather(buf, base, stride, rows, cols):
    """interp._tile_gather (interp.py:408-410): buf[base + i*stride + j]."""
    idx = base + stride * np.arange(rows)[:, None] + np.arange(cols)[None, :]
    buf = np.asarray(buf)
    if idx.min() < 0 or idx.max() >= len(buf):
        raise IndexError("tile gather out of bounds")
    return buf[idx.reshape(-1)]


def window_times_matrix(window, mat):
    """test_layout.window_times_matrix: out[x] = sum_y window[y]*A[y][x], left to right."""
    window = np.asarray(window, np.float32)
    mat = np.asarray(mat, np.float32)
    return foldl_rows((window[:, None] * mat).T)
