"""ctypes binding of the sm_100a native library (include/tensorsel_b200.h).

The library is built in-tree (``paper_2512_02371_b200/_native/libtsb200.so``)
by ``__graft_entry__.build()`` / ``python -m paper_2512_02371_b200.build``.
There is no fallback: if the library is missing every product entry point
raises :class:`NativeLibraryMissing`.
"""

from __future__ import annotations

import ctypes
import os
import threading

from . import errors

_HERE = os.path.dirname(os.path.abspath(__file__))
# TSB_LIB_PATH: an alternative build of the same library (same-box A/B experiments)
LIB_PATH = os.environ.get("TSB_LIB_PATH") or os.path.join(_HERE, "_native", "libtsb200.so")

TS_BF16, TS_F32, TS_F16 = 1, 2, 3
ABI_VERSION = 2  # include/tensorsel_b200.h TS_ABI_VERSION
TS_AXIS_DC_EXACT = 0x1

_lock = threading.Lock()
_lib = None
_diag = None


class ConvGroup(ctypes.Structure):
    """ts_conv_group (include/tensorsel_b200.h)."""
    _fields_ = [
        ("instances", ctypes.c_int),
        ("src", ctypes.c_void_p), ("src_stride", ctypes.c_int64),
        ("src_len", ctypes.c_int), ("src_kind", ctypes.c_int),
        ("kern", ctypes.c_void_p), ("kern_stride", ctypes.c_int64),
        ("kern_len", ctypes.c_int), ("kern_kind", ctypes.c_int),
        ("acc", ctypes.c_void_p), ("acc_stride", ctypes.c_int64), ("zero_init", ctypes.c_int),
        ("m", ctypes.c_int), ("k", ctypes.c_int), ("n", ctypes.c_int), ("a_stride", ctypes.c_int),
        ("iterations", ctypes.c_int),
        ("a_base", ctypes.c_void_p), ("k_base", ctypes.c_void_p), ("b_off", ctypes.c_void_p),
        ("a_idx", ctypes.c_void_p), ("b_idx", ctypes.c_void_p),
        ("error", ctypes.c_void_p),
        ("a_shift", ctypes.c_void_p),
        ("out_base", ctypes.c_void_p), ("out_off", ctypes.c_void_p),
        ("out", ctypes.c_void_p), ("out_stride", ctypes.c_int64),
    ]


class AxisInfo(ctypes.Structure):
    _fields_ = [(n, ctypes.c_int) for n in (
        "n_in", "n_out", "taps", "window", "blocks", "unique_tiles",
        "row_span", "col_blocks", "col_span")]

    def as_dict(self):
        return {n: getattr(self, n) for n, _ in self._fields_}


class Epilogue(ctypes.Structure):
    """ts_epilogue: y = min(max(x * scale + bias, lo), hi), inside the kernel."""
    _fields_ = [("scale", ctypes.c_float), ("bias", ctypes.c_float),
                ("lo", ctypes.c_float), ("hi", ctypes.c_float)]


_P = ctypes.c_void_p
_I = ctypes.c_int
_I64 = ctypes.c_int64
_FP = ctypes.POINTER(ctypes.c_float)
_IP = ctypes.POINTER(ctypes.c_int32)

# name -> (restype, argtypes)
_SIGNATURES = {
    "ts_last_error": (ctypes.c_char_p, []),
    "ts_abi_version": (_I, []),
    "ts_device_count": (_I, []),
    "ts_axis_create": (_I, [_I, _I, _I, _IP, _FP, _I, _I, ctypes.POINTER(_P)]),
    "ts_axis_from_toeplitz": (_I, [_I, _I, _I, _I, _FP, _I, _I, _I, _I, _I,
                                   ctypes.POINTER(_P)]),
    "ts_axis_get_info": (_I, [_P, ctypes.POINTER(AxisInfo)]),
    "ts_axis_dense": (_I, [_P, _FP]),
    "ts_axis_destroy": (None, [_P]),
    "ts_separable_run": (_I, [_P, _P, _I, _P, _I64, _I64, _I, _P, _I64, _I64, _I, _P]),
    "ts_separable_run_ep": (_I, [_P, _P, _I, _P, _I64, _I64, _I, _P, _I64, _I64, _I,
                                 ctypes.POINTER(Epilogue), _P]),
    "ts_separable_plan": (_I, [_P, _P, _I, _I, ctypes.POINTER(ctypes.c_int)]),
    "ts_axis_pass": (_I, [_P, _I, _I, _I, _I, _P, _I64, _I64, _P, _I64, _I64, _I, _P]),
    "ts_axis_pass_ep": (_I, [_P, _I, _I, _I, _I, _P, _I64, _I64, _P, _I64, _I64, _I,
                             ctypes.POINTER(Epilogue), _P]),
    "ts_cast_f32_bf16": (_I, [_P, _P, _I64, _P]),
    "ts_separable_f32_ep": (_I, [_I, _P, _I, _I, _I64, _I64, _I, _I, _I, _P, _I, _I, _P, _I, _P,
                                 _I64, _I64, _I, _I, _P, _P]),
    "ts_run_conv_group": (_I, [_P, _P]),
    "ts_denoise_dct16": (_I, [_P, _I64, _I64, _I, _P, _I64, _I64, _I, _I, _I, _I,
                              ctypes.c_float, _I, _P]),
    "ts_denoise_dct16_ep": (_I, [_P, _I64, _I64, _I, _P, _I64, _I64, _I, _I, _I, _I,
                                 ctypes.c_float, _I, ctypes.POINTER(Epilogue), _P]),
    "ts_matrix_for": (_I, [_I, _I, _I, _I, _P, _P, _P]),
}

EXPORTED = tuple(_SIGNATURES)

# Diagnostics (tools only): libtsb200_diag.so = the product sources built with
# -DTSB_DIAG plus tools/diag/probe.cu; declared in tools/diag/tsb_diag.h.
DIAG_LIB_PATH = os.path.join(_HERE, "_native", "libtsb200_diag.so")
_DIAG_SIGNATURES = {
    "ts_probe_tma": (_I, [_P, _I, _I, _I, _I, _I, _I, _I, _P]),
    "ts_probe_tmem_ld": (_I, [_I, _I, _I, _I, _P, _P]),
    "ts_probe_m64": (_I, [_P, _P, _P, _I, _I, _P]),
    "ts_probe_issue2": (_I, [_I, _I, _I, _I, _I, _P, _P]),
    "ts_debug_dct16": (_I, [_P]),
    "ts_probe_umma": (_I, [_P, _P, _P, _I, _I, _P]),
    "ts_debug_trace": (_I, [_P, _I, _I]),
    "ts_probe_mma": (_I, [_I, _I, _P, _P, _P, _I, _I, _I, _P, _I, _P]),
    "ts_probe_issue": (_I, [_I, _P, _P]),
    "ts_probe_issue_ts": (_I, [_I, _P, _P]),
}


class NativeLibraryMissing(RuntimeError):
    pass


def load(path: str | None = None):
    """Load (once) and return the native library handle."""
    global _lib
    with _lock:
        if _lib is not None and path is None:
            return _lib
        p = path or LIB_PATH
        if not os.path.exists(p):
            raise NativeLibraryMissing(
                f"native library not built: {p} (run `python -m paper_2512_02371_b200.build`)")
        lib = ctypes.CDLL(p)
        for name, (res, args) in _SIGNATURES.items():
            fn = getattr(lib, name)
            fn.restype = res
            fn.argtypes = args
        if lib.ts_abi_version() != ABI_VERSION:
            raise NativeLibraryMissing(f"ABI mismatch: library reports {lib.ts_abi_version()}")
        if path is None:
            _lib = lib
        return lib


def load_diag():
    """The diagnostics library (``make -C paper_2512_02371_b200/csrc diag``):
    every product entry point plus trace hooks and micro-probes.  Tools
    only; the product never loads it."""
    global _diag
    if os.path.abspath(LIB_PATH) == os.path.abspath(DIAG_LIB_PATH):
        load()  # TSB_LIB_PATH points the product binding at the diag build (trace tools)
    with _lock:
        if _diag is None and _lib is not None and \
                os.path.abspath(LIB_PATH) == os.path.abspath(DIAG_LIB_PATH):
            for name, (res, args) in _DIAG_SIGNATURES.items():
                fn = getattr(_lib, name)
                fn.restype = res
                fn.argtypes = args
            _diag = _lib
        if _diag is None:
            if not os.path.exists(DIAG_LIB_PATH):
                raise NativeLibraryMissing(
                    f"diagnostics library not built: {DIAG_LIB_PATH} "
                    "(run `make -C paper_2512_02371_b200/csrc diag`)")
            lib = ctypes.CDLL(DIAG_LIB_PATH)
            for name, (res, args) in {**_SIGNATURES, **_DIAG_SIGNATURES}.items():
                fn = getattr(lib, name)
                fn.restype = res
                fn.argtypes = args
            _diag = lib
        return _diag


def last_error() -> str:
    msg = load().ts_last_error()
    return msg.decode() if msg else ""


def check(status: int, what: str = "") -> None:
    """Raise the reference-compatible exception for a non-OK ts_status."""
    if status == 0:
        return
    msg = last_error()
    if what:
        msg = f"{what}: {msg}"
    raise errors.from_status(status, msg)
