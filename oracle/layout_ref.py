"""Restated Toeplitz-family builders, plain loop form.

TEST INFRASTRUCTURE ONLY.  Restates /root/reference/pkg/src/tensorsel/layout.py
so the product module (paper_2512_02371_b200/layout.py, vectorised) and the
device builder can be checked against an independent implementation.
"""

from __future__ import annotations

import numpy as np


class PhaseMismatch(Exception):
    pass


def rows_for(l, k, s=1, p=1):
    """layout.matrix_rows (layout.py:54-57)."""
    return k // p + l if p > 1 else s * k + l


def tap_at(l, s, p, y, x):
    """layout.kernel_taps (layout.py:60-69)."""
    if p > 1:
        u = y - x // p
        return p * u + x % p if 0 <= u < l else None
    t = y - s * x
    return t if 0 <= t < l else None


def dense(kernel, l, k, s=1, p=1):
    """layout.matrix_for (layout.py:72-84)."""
    kernel = np.asarray(kernel)
    if len(kernel) != p * l:
        raise PhaseMismatch(f"kernel has {len(kernel)} taps, spec needs {p * l}")
    out = np.zeros((rows_for(l, k, s, p), k), dtype=kernel.dtype)
    for y in range(out.shape[0]):
        for x in range(k):
            t = tap_at(l, s, p, y, x)
            if t is not None:
                out[y, x] = kernel[t]
    return out


def shuffle_indices(l, k, s, p, base, buffer_length):
    """layout.shuffle_indices_for (layout.py:106-122)."""
    if base < 0 or base + p * l > buffer_length:
        raise IndexError("kernel window exceeds buffer")
    out = []
    for y in range(rows_for(l, k, s, p)):
        for x in range(k):
            t = tap_at(l, s, p, y, x)
            out.append(-1 if t is None else t + 1)
    return out


def banded_axis(n_in, first, weights):
    """Dense n_out x n_in matrix of an axis (output o reads inputs
    first[o] + t with weights[o, t]), indices clamped to the edge."""
    first = np.asarray(first)
    weights = np.asarray(weights, np.float64)
    n_out, taps = weights.shape
    m = np.zeros((n_out, n_in), np.float64)
    for o in range(n_out):
        for t in range(taps):
            i = min(max(int(first[o]) + t, 0), n_in - 1)
            m[o, i] += weights[o, t]
    return m
