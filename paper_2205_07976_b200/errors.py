"""Error types of the spot path, named as in the reference.

The reference's hierarchy lives in /root/reference/pkg/src/xtrace/errors.py:4-61;
the spot kernel raises ShapeMismatchError (kernels.py:204-208) and, for a
non-finite pixel, NumericalFault wrapped in PatternFault (kernels.py:211-216,
execution.py:183-185,217-224).  Callers that catch the reference's classes by
name (or by their builtin bases ValueError / ArithmeticError / RuntimeError)
keep working.
"""
from __future__ import annotations

import sys
from types import ModuleType

__all__ = [
    "XtraceError",
    "InvalidCellError",
    "GeometryError",
    "OutOfBoundsError",
    "ShapeMismatchError",
    "NumericalFault",
    "PatternFault",
    "NativeError",
    "CampaignIOError",
    "hierarchy_for",
]


class XtraceError(Exception):
    """Root of every error raised by this package."""


class InvalidCellError(XtraceError, ValueError):
    """Cell edges/angles that do not span a lattice."""


class GeometryError(XtraceError, ValueError):
    """Detector, beam or rotation geometry that is degenerate or not unit/orthonormal."""


class OutOfBoundsError(XtraceError, IndexError):
    """A pixel or domain index outside its grid."""


class ShapeMismatchError(XtraceError, ValueError):
    """Buffer dims or precision do not match what the kernel needs."""


class NumericalFault(XtraceError, ArithmeticError):
    """A pixel evaluated to a non-finite value; ``pixel`` is its flat index."""

    def __init__(self, pixel: int, message: str = ""):
        self.pixel = int(pixel)
        super().__init__(message or f"non-finite value at pixel {self.pixel}")


class PatternFault(XtraceError, RuntimeError):
    """A kernel launch failed at ``index`` (the lowest failing pixel); ``cause`` says why."""

    def __init__(self, label: str, index: int, cause: BaseException):
        self.label = label
        self.index = int(index)
        self.cause = cause
        super().__init__(f"pattern {label!r} failed at index {self.index}: {cause!r}")


class CampaignIOError(XtraceError, OSError):
    """Writing a campaign image failed (errors.py:55-61 of the reference); carries the image index."""

    def __init__(self, image_index: int, cause):
        self.image_index = int(image_index)
        self.cause = cause
        super().__init__(f"I/O failure on image {self.image_index}: {cause}")


class NativeError(XtraceError, RuntimeError):
    """The CUDA library is missing, found no GPU, or a CUDA call failed.

    There is deliberately no CPU fallback: the product path fails loudly.
    """


def hierarchy_for(*objs) -> ModuleType:
    """The module whose error classes a call on ``objs`` raises.

    When the inputs are the reference's own objects (``xtrace.kernels.SpotsContext``,
    ``xtrace.kernels.PixelBuffer``, ...) the drop-in raises the reference's classes
    (``xtrace.errors.ShapeMismatchError`` / ``PatternFault`` / ``NumericalFault``,
    errors.py:20-39 of the reference), so ``except (NumericalFault, PatternFault)`` in the
    reference's own callers (scheduler.py:212) catches them; otherwise this module's.
    """
    for o in objs:
        top = type(o).__module__.partition(".")[0]
        if not top or top == __name__.partition(".")[0]:
            continue
        mod = sys.modules.get(top + ".errors")
        if mod is not None and all(hasattr(mod, n) for n in ("ShapeMismatchError", "NumericalFault",
                                                              "PatternFault")):
            return mod
    return sys.modules[__name__]
