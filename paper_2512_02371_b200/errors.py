"""Exception classes mirroring the reference's error surface.

``interp.EvalError`` and its subclasses (interp.py:32-55) and
``layout.PhaseMismatch`` / ``layout.OutOfBounds`` (layout.py:24-29) are the
reference's error vocabulary; the native library reports the same conditions
as ``ts_status`` codes which :func:`from_status` maps back.
"""

from __future__ import annotations

# Interoperability with the reference: when the reference package is
# importable next to this one (the drop-in case), every class below also
# derives from its reference counterpart, so a caller's
# ``except tensorsel.interp.OutOfBounds`` catches this package's errors too.
try:  # pragma: no cover - depends on the caller's environment
    from tensorsel import interp as _ref_interp, layout as _ref_layout
except Exception:  # the reference is optional
    _ref_interp = _ref_layout = None


def _ref(mod, name):
    return (getattr(mod, name),) if mod is not None and hasattr(mod, name) else ()


class EvalError(*_ref(_ref_interp, "EvalError"), Exception):
    """interp.EvalError (interp.py:32)."""


class OutOfBounds(EvalError, *_ref(_ref_interp, "OutOfBounds")):
    """interp.OutOfBounds (interp.py:36-39)."""

    def __init__(self, buffer, index=None):
        if index is None:  # message-only form from the native layer
            Exception.__init__(self, buffer)
            self.buffer, self.index = None, None
        else:
            Exception.__init__(self, f"buffer {buffer!r} index {index} out of bounds")
            self.buffer, self.index = buffer, index


class DivideByZero(EvalError, *_ref(_ref_interp, "DivideByZero")):
    """interp.DivideByZero (interp.py:42)."""


class UnknownIntrinsic(EvalError, *_ref(_ref_interp, "UnknownIntrinsic")):
    """interp.UnknownIntrinsic (interp.py:46)."""


class ShapeUnregistered(EvalError, *_ref(_ref_interp, "ShapeUnregistered")):
    """interp.ShapeUnregistered (interp.py:50)."""


class I32Overflow(EvalError, *_ref(_ref_interp, "I32Overflow")):
    """interp.I32Overflow (interp.py:54)."""


class PhaseMismatch(*_ref(_ref_layout, "PhaseMismatch"), Exception):
    """layout.PhaseMismatch (layout.py:24)."""


class LayoutOutOfBounds(*_ref(_ref_layout, "OutOfBounds"), Exception):
    """layout.OutOfBounds (layout.py:28)."""


class UnsupportedGeometry(EvalError):
    """A shape the sm_100a kernels cannot tile (no reference counterpart)."""


class CudaError(RuntimeError):
    """A CUDA runtime/driver failure inside the native library."""


class NoDevice(RuntimeError):
    """No sm_100 device is visible."""


_BY_STATUS = {
    1: EvalError,
    2: OutOfBounds,
    3: PhaseMismatch,
    4: ShapeUnregistered,
    5: UnknownIntrinsic,
    6: UnsupportedGeometry,
    7: CudaError,
    8: NoDevice,
}


def from_status(status: int, msg: str) -> Exception:
    cls = _BY_STATUS.get(status, EvalError)
    return cls(msg)
