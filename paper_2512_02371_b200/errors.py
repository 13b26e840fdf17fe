"""Exception classes mirroring the reference's error surface.

``interp.EvalError`` and its subclasses (interp.py:32-55) and
``layout.PhaseMismatch`` / ``layout.OutOfBounds`` (layout.py:24-29) are the
reference's error vocabulary; the native library reports the same conditions
as ``ts_status`` codes which :func:`from_status` maps back.
"""

from __future__ import annotations


class EvalError(Exception):
    """interp.EvalError (interp.py:32)."""


class OutOfBounds(EvalError):
    """interp.OutOfBounds (interp.py:36-39)."""

    def __init__(self, buffer, index=None):
        if index is None:  # message-only form from the native layer
            super().__init__(buffer)
            self.buffer, self.index = None, None
        else:
            super().__init__(f"buffer {buffer!r} index {index} out of bounds")
            self.buffer, self.index = buffer, index


class DivideByZero(EvalError):
    """interp.DivideByZero (interp.py:42)."""


class UnknownIntrinsic(EvalError):
    """interp.UnknownIntrinsic (interp.py:46)."""


class ShapeUnregistered(EvalError):
    """interp.ShapeUnregistered (interp.py:50)."""


class I32Overflow(EvalError):
    """interp.I32Overflow (interp.py:54)."""


class PhaseMismatch(Exception):
    """layout.PhaseMismatch (layout.py:24)."""


class LayoutOutOfBounds(Exception):
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
