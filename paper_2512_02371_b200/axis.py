"""Device-resident banded axis matrices (the weight-matrix builder's output).

An :class:`Axis` is one side of a separable linear transform: the banded
``n_out x n_in`` matrix of a resample or filter, with clamp-to-edge folded
in, built by the native builder (csrc/builder.cpp) into 16-output blocks of
bf16 tcgen05 B-operand tiles.  Building is the analogue of the reference's
ExprVar hoisting (selector.py:309-399): it happens once per
(kernel, scale, size, device) and is cached.
"""

from __future__ import annotations

import ctypes
import threading

import numpy as np

from . import _lib, filters, layout


class Axis:
    def __init__(self, n_in: int, n_out: int, first, weights, *, device: int = 0,
                 dc_exact: bool = True):
        first = np.ascontiguousarray(first, dtype=np.int32)
        weights = np.ascontiguousarray(weights, dtype=np.float32)
        if weights.ndim != 2 or weights.shape[0] != n_out or first.shape != (n_out,):
            raise ValueError(f"weights must be ({n_out}, taps) and first ({n_out},)")
        lib = _lib.load()
        h = ctypes.c_void_p()
        st = lib.ts_axis_create(
            int(n_in), int(n_out), int(weights.shape[1]),
            first.ctypes.data_as(ctypes.POINTER(ctypes.c_int32)),
            weights.ctypes.data_as(ctypes.POINTER(ctypes.c_float)),
            _lib.TS_AXIS_DC_EXACT if dc_exact else 0, int(device), ctypes.byref(h))
        _lib.check(st, "ts_axis_create")
        self._h = h
        self.device = device
        self.n_in, self.n_out = int(n_in), int(n_out)
        self.info = self._info()
        self.first, self.weights = first, weights  # f32 taps (the FMA-pipe f32 path)

    @property
    def uniform(self):
        """(stride, taps, base) when output o reads inputs stride*o + base + t
        with the same taps for every o (the f32 kernel's precondition), else
        None."""
        first = getattr(self, "first", None)
        if first is None or self.n_out < 1:
            return None
        base = int(first[0])
        stride = int(first[1] - first[0]) if self.n_out > 1 else 1
        if stride < 1 or not np.array_equal(
                first, base + stride * np.arange(self.n_out, dtype=np.int64)):
            return None
        if not (self.weights == self.weights[:1]).all():
            return None
        return stride, int(self.weights.shape[1]), base

    def device_weights(self):
        """The f32 taps as a device tensor (n_out x taps), uploaded once."""
        w = getattr(self, "_wdev", None)
        if w is None:
            import torch
            w = self._wdev = torch.from_numpy(self.weights).to(f"cuda:{self.device}")
        return w

    @classmethod
    def from_toeplitz(cls, spec: layout.ToeplitzSpec, kernel, n_in: int, n_out: int,
                      offset: int = 0, *, device: int = 0, dc_exact: bool = False):
        """Axis whose blocks are the reference Toeplitz-family matrix of
        ``spec`` (layout.py:32-103), first tap at ``offset``."""
        kernel = np.ascontiguousarray(kernel, dtype=np.float32)
        lib = _lib.load()
        h = ctypes.c_void_p()
        st = lib.ts_axis_from_toeplitz(
            spec.l, spec.s, spec.p, int(offset),
            kernel.ctypes.data_as(ctypes.POINTER(ctypes.c_float)), len(kernel),
            int(n_in), int(n_out), _lib.TS_AXIS_DC_EXACT if dc_exact else 0, int(device),
            ctypes.byref(h))
        _lib.check(st, "ts_axis_from_toeplitz")
        self = cls.__new__(cls)
        self._h = h
        self.device = device
        self.n_in, self.n_out = int(n_in), int(n_out)
        self.info = self._info()
        return self

    def _info(self):
        info = _lib.AxisInfo()
        _lib.check(_lib.load().ts_axis_get_info(self._h, ctypes.byref(info)), "ts_axis_get_info")
        return info.as_dict()

    @property
    def handle(self):
        return self._h

    def dense(self) -> np.ndarray:
        """The effective (bf16-rounded, edge-folded) n_out x n_in matrix."""
        out = np.zeros((self.n_out, self.n_in), dtype=np.float32)
        _lib.check(_lib.load().ts_axis_dense(
            self._h, out.ctypes.data_as(ctypes.POINTER(ctypes.c_float))), "ts_axis_dense")
        return out

    def __del__(self):
        h = getattr(self, "_h", None)
        if h is not None and h.value:
            try:
                _lib.load().ts_axis_destroy(h)
            except Exception:
                pass
            self._h = None


_cache: dict = {}
_cache_lock = threading.Lock()


def cached(key, build):
    with _cache_lock:
        a = _cache.get(key)
    if a is None:
        a = build()
        with _cache_lock:
            _cache.setdefault(key, a)
            a = _cache[key]
    return a


def lanczos3(n_in: int, n_out: int, device: int) -> Axis:
    def build():
        first, w = filters.lanczos3_axis(n_in, n_out)
        return Axis(n_in, n_out, first, w, device=device)
    return cached(("lanczos3", n_in, n_out, device), build)


def convolution(n: int, kernel, device: int) -> Axis:
    kernel = np.asarray(kernel, dtype=np.float32)
    def build():
        first, w = filters.conv_axis(n, kernel)
        return Axis(n, n, first, w, device=device)
    return cached(("conv", n, kernel.tobytes(), device), build)


def resample_filter(n_in: int, n_mid: int, kernel, device: int) -> Axis:
    """Lanczos-3 resample n_in -> n_mid followed by a same-size centred
    filter, composed into one banded axis (config 5 runs as ONE pass)."""
    from . import partition
    kernel = np.asarray(kernel, dtype=np.float32)

    def build():
        inner = filters.lanczos3_axis(n_in, n_mid)
        outer = filters.conv_axis(n_mid, kernel)
        first, w = partition.compose_axes(outer, inner, n_mid, n_in)
        return Axis(n_in, n_mid, first, w, device=device)
    return cached(("lanczos+conv", n_in, n_mid, kernel.tobytes(), device), build)
