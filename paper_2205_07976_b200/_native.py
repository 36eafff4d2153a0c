"""ctypes binding of the C ABI in include/nbx.h (libnbx.so, built in-tree).

The library is the product: there is no CPU fallback.  If the .so is missing
or no GPU is visible, every entry point raises NativeError with the reason.
ctypes releases the GIL for the duration of each call.
"""
from __future__ import annotations

import ctypes as C
import os
import sys
import threading
from pathlib import Path

import numpy as np

from .errors import NativeError

LIB_PATH = Path(os.environ.get("NBX_LIB") or Path(__file__).resolve().parent / "_lib" / "libnbx.so")

NBX_OK, NBX_ERR_ARG, NBX_ERR_NUMERICAL, NBX_ERR_CUDA, NBX_ERR_IO = 0, 1, 2, 3, 4
COMPUTE = {"fp64": 0, "fp32": 1}
OUT_F32, OUT_F64, OUT_ADD_F64, OUT_RAW_F64, OUT_IMAGE_F64, OUT_IMAGE_F32, OUT_RAW_STORE_F64 = 0, 1, 2, 3, 4, 5, 6
SHAPES = {"sincg": 0, "square": 0, "gauss": 1, "round": 2, "tophat": 3}

# Every exported symbol of include/nbx.h (checked by tests/test_abi.py).
EXPORTS = (
    "nbx_version", "nbx_ctx_create", "nbx_ctx_destroy", "nbx_last_error", "nbx_ctx_set_stream",
    "nbx_ctx_synchronize", "nbx_output_pixels", "nbx_spots", "nbx_spots_batch", "nbx_plan_create",
    "nbx_plan_run", "nbx_plan_info", "nbx_plan_last_kernel_ms", "nbx_plan_destroy", "nbx_finalize",
    "nbx_add_array", "nbx_add_noise", "nbx_poisson_host", "nbx_probe_fma_peak", "nbx_background",
    "nbx_fault_stage", "nbx_spots_reduce", "nbx_campaign", "nbx_crc32", "nbx_image_stats", "nbx_image_histogram",
    "nbx_struct_size", "nbx_device_count", "nbx_ipc_alloc", "nbx_ipc_free", "nbx_ipc_open", "nbx_ipc_close", "nbx_reduce_slots",
)


class Panel(C.Structure):
    _fields_ = [
        ("slow_pixels", C.c_int32), ("fast_pixels", C.c_int32), ("thick_steps", C.c_int32),
        ("reserved0", C.c_int32), ("pixel_size", C.c_double), ("distance", C.c_double),
        ("beam_center", C.c_double * 2), ("fast_axis", C.c_double * 3), ("slow_axis", C.c_double * 3),
        ("thickness", C.c_double), ("attenuation_length", C.c_double),
    ]


class SpotsDesc(C.Structure):
    _fields_ = [
        ("n_panels", C.c_int32), ("oversample", C.c_int32), ("panels", C.POINTER(Panel)),
        ("beam_direction", C.c_double * 3), ("polarization_on", C.c_int32), ("n_sources", C.c_int32),
        ("wavelengths", C.POINTER(C.c_double)), ("weights", C.POINTER(C.c_double)),
        ("fluence", C.c_double), ("r_e_sqr", C.c_double),
        ("n_domains", C.c_int32), ("shape", C.c_int32), ("bases", C.POINTER(C.c_double)),
        ("n_cells", C.c_int32 * 3), ("n_entries", C.c_int32), ("hkl", C.POINTER(C.c_int32)),
        ("amplitudes", C.POINTER(C.c_double)), ("default_f", C.c_double), ("norm", C.c_double),
        ("src_begin", C.c_int32), ("src_end", C.c_int32),
        ("bg_points", C.c_int32), ("reserved1", C.c_int32), ("bg_stol", C.POINTER(C.c_double)),
        ("bg_f", C.POINTER(C.c_double)), ("bg_thickness_factor", C.c_double),
    ]


class PlanInfo(C.Structure):
    _fields_ = [
        ("n_pixels", C.c_int64), ("steps", C.c_int64), ("table_cells", C.c_int64),
        ("table_lo", C.c_int32 * 3), ("table_dim", C.c_int32 * 3), ("compute", C.c_int32),
        ("table_kind", C.c_int32), ("scale", C.c_double), ("channel_runs", C.c_int32), ("kernel_variant", C.c_int32),
    ]


_lib = None
_lock = threading.RLock()


def load() -> C.CDLL:
    """Load libnbx.so once; raise NativeError if it is absent."""
    global _lib
    if _lib is not None:
        return _lib
    with _lock:
        if _lib is not None:
            return _lib
        if not LIB_PATH.exists():
            raise NativeError(f"native library missing: {LIB_PATH} (run `python -m paper_2205_07976_b200.build`)")
        lib = C.CDLL(str(LIB_PATH))
        vp, i64p = C.c_void_p, C.POINTER(C.c_int64)
        sig = {
            "nbx_version": (C.c_int, []),
            "nbx_ctx_create": (vp, [C.c_int]),
            "nbx_ctx_destroy": (None, [vp]),
            "nbx_last_error": (C.c_char_p, [vp]),
            "nbx_ctx_set_stream": (C.c_int, [vp, vp]),
            "nbx_ctx_synchronize": (C.c_int, [vp]),
            "nbx_output_pixels": (C.c_int64, [C.POINTER(SpotsDesc)]),
            "nbx_spots": (C.c_int, [vp, C.POINTER(SpotsDesc), C.c_int, C.c_int, vp, C.c_int, i64p]),
            "nbx_spots_batch": (C.c_int, [vp, C.POINTER(SpotsDesc), C.c_int, C.c_int, C.c_int,
                                          C.POINTER(vp), C.c_int, i64p]),
            "nbx_plan_create": (vp, [vp, C.POINTER(SpotsDesc), C.c_int]),
            "nbx_plan_run": (C.c_int, [vp, C.c_int, vp, C.c_int, i64p]),
            "nbx_plan_info": (C.c_int, [vp, C.POINTER(PlanInfo)]),
            "nbx_plan_last_kernel_ms": (C.c_double, [vp]),
            "nbx_plan_destroy": (None, [vp]),
            "nbx_finalize": (C.c_int, [vp, vp, C.c_int64, C.c_double, C.c_int, vp, C.c_int, i64p]),
            "nbx_add_array": (C.c_int, [vp, vp, vp, C.c_int64, C.c_int]),
            "nbx_add_noise": (C.c_int, [vp, vp, vp, C.c_int64, C.c_int, C.c_uint64, C.c_uint64, C.c_int]),
            "nbx_poisson_host": (C.c_int, [vp, vp, C.c_int64, C.c_int, C.c_uint64, C.c_uint64]),
            "nbx_probe_fma_peak": (C.c_int, [vp, C.c_int, C.POINTER(C.c_double)]),
            "nbx_background": (C.c_int, [vp, C.POINTER(SpotsDesc), C.c_int, vp, C.c_int, i64p]),
            "nbx_fault_stage": (C.c_int, [vp]),
            "nbx_spots_reduce": (C.c_int, [vp, C.POINTER(SpotsDesc), C.c_int, vp, C.c_int, C.c_int, vp, C.c_int,
                                           i64p]),
            "nbx_campaign": (C.c_int, [vp, C.POINTER(SpotsDesc), C.c_int, C.c_int, C.POINTER(C.c_char_p),
                                       C.POINTER(C.c_uint32), i64p]),
            "nbx_crc32": (C.c_uint32, [C.c_uint32, vp, C.c_int64]),
            "nbx_image_stats": (C.c_int, [vp, vp, C.c_int64, C.c_int, C.c_int, C.POINTER(C.c_double)]),
            "nbx_image_histogram": (C.c_int, [vp, vp, C.c_int64, C.c_int, C.c_int, C.c_int, C.c_double,
                                              C.c_double, i64p, i64p, i64p]),
            "nbx_struct_size": (C.c_int64, [C.c_int]),
            "nbx_device_count": (C.c_int, []),
            "nbx_ipc_alloc": (C.c_int, [vp, C.c_int64, C.POINTER(vp), C.c_char_p]),
            "nbx_ipc_free": (C.c_int, [vp, vp]),
            "nbx_ipc_open": (C.c_int, [vp, C.c_char_p, C.POINTER(vp)]),
            "nbx_ipc_close": (C.c_int, [vp, vp]),
            "nbx_reduce_slots": (C.c_int, [vp, vp, C.c_int, C.c_int64, C.c_double, C.c_int, vp, C.c_int, i64p]),
        }
        for name, (res, args) in sig.items():
            fn = getattr(lib, name)
            fn.restype = res
            fn.argtypes = args
        _lib = lib
        return lib


def default_device() -> int:
    """Device of the default context: NBX_DEVICE if set; else torch's current device once torch
    has initialised CUDA (``torch.cuda.set_device(local_rank)``); else LOCAL_RANK under torchrun
    (one process per GPU, wrapped onto the visible devices); else 0."""
    env = os.environ.get("NBX_DEVICE")
    if env is not None:
        return int(env)
    torch = sys.modules.get("torch")
    if torch is not None and torch.cuda.is_initialized():
        return int(torch.cuda.current_device())
    local = os.environ.get("LOCAL_RANK")
    if local is not None:
        n = load().nbx_device_count()
        return int(local) % n if n > 0 else 0
    return 0


class Context:
    """One CUDA device: stream, events, scratch (nbx_ctx_create)."""

    def __init__(self, device: int | None = None):
        self.lib = load()
        # The C ABI serves one host thread at a time per context (include/nbx.h); ctypes drops
        # the GIL during calls, so every call that touches this context's streams / scratch and
        # the status check that reads its last-error string happen under this lock.
        self.lock = threading.RLock()
        self.device = default_device() if device is None else int(device)
        self.handle = self.lib.nbx_ctx_create(self.device)
        if not self.handle:
            raise NativeError(f"nbx_ctx_create({self.device}) failed: "
                              f"{self.lib.nbx_last_error(None).decode(errors='replace')}")

    def error(self) -> str:
        return self.lib.nbx_last_error(self.handle).decode(errors="replace")

    def close(self):
        if getattr(self, "handle", None):
            self.lib.nbx_ctx_destroy(self.handle)
            self.handle = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


_contexts: dict[int, Context] = {}


def context(device: int | None = None) -> Context:
    dev = default_device() if device is None else int(device)
    ctx = _contexts.get(dev)
    if ctx is None:
        with _lock:
            ctx = _contexts.get(dev)
            if ctx is None:
                ctx = Context(dev)
                _contexts[dev] = ctx
    return ctx


def ptr(arr: np.ndarray, ctype):
    return arr.ctypes.data_as(C.POINTER(ctype))


class Descriptor:
    """A filled SpotsDesc plus the NumPy arrays that back its pointers."""

    def __init__(self, *, panels, oversample, beam_direction, polarization_on, wavelengths, weights,
                 fluence, r_e_sqr, bases, n_cells, hkl, amplitudes, default_f, shape=0, norm=0.0,
                 src_begin=0, src_end=0, background=None, thickness_factor=1.0):
        self._panels = (Panel * len(panels))()
        for dst, p in zip(self._panels, panels):
            dst.slow_pixels = int(p.slow_pixels)
            dst.fast_pixels = int(p.fast_pixels)
            dst.thick_steps = int(getattr(p, "thick_steps", 1))
            dst.pixel_size = float(p.pixel_size)
            dst.distance = float(p.distance)
            dst.beam_center[:] = [float(x) for x in p.beam_center]
            dst.fast_axis[:] = [float(x) for x in p.fast_axis]
            dst.slow_axis[:] = [float(x) for x in p.slow_axis]
            dst.thickness = float(getattr(p, "thickness", 0.0))
            dst.attenuation_length = float(getattr(p, "attenuation_length", 0.0))
        self._wl = np.ascontiguousarray(wavelengths, dtype=np.float64)
        self._w = np.ascontiguousarray(weights, dtype=np.float64)
        self._bases = np.ascontiguousarray(bases, dtype=np.float64).reshape(-1, 3, 3)
        self._hkl = np.ascontiguousarray(hkl, dtype=np.int32).reshape(-1, 3)
        self._amp = np.ascontiguousarray(amplitudes, dtype=np.float64).reshape(-1)
        d = SpotsDesc()
        d.n_panels = len(panels)
        d.oversample = int(oversample)
        d.panels = C.cast(self._panels, C.POINTER(Panel))
        d.beam_direction[:] = [float(x) for x in beam_direction]
        d.polarization_on = 1 if polarization_on else 0
        d.n_sources = self._wl.size
        d.wavelengths = ptr(self._wl, C.c_double)
        d.weights = ptr(self._w, C.c_double)
        d.fluence = float(fluence)
        d.r_e_sqr = float(r_e_sqr)
        d.n_domains = self._bases.shape[0]
        d.shape = int(shape)
        d.bases = ptr(self._bases, C.c_double)
        d.n_cells[:] = [int(x) for x in n_cells]
        d.n_entries = self._hkl.shape[0]
        d.hkl = ptr(self._hkl, C.c_int32)
        d.amplitudes = ptr(self._amp, C.c_double)
        d.default_f = float(default_f)
        d.norm = float(norm)
        d.src_begin = int(src_begin)
        d.src_end = int(src_end)
        if background is not None:  # BackgroundProfile (model.py:409-435)
            self._bg_stol = np.ascontiguousarray(background.stol, dtype=np.float64)
            self._bg_f = np.ascontiguousarray(background.f_bg, dtype=np.float64)
            d.bg_points = self._bg_stol.size
            d.bg_stol = ptr(self._bg_stol, C.c_double)
            d.bg_f = ptr(self._bg_f, C.c_double)
            d.bg_thickness_factor = float(thickness_factor)
        self.c = d

    @property
    def n_pixels(self) -> int:
        return sum(int(p.slow_pixels) * int(p.fast_pixels) for p in self._panels)


def check(ctx: Context, status: int, first_bad: int = -1, label: str = "nanobragg_spots", errors=None):
    """Translate an NBX status into the reference's exceptions.

    ``errors`` is the module whose classes are raised (``errors.hierarchy_for``: the
    reference's own ``xtrace.errors`` when the call came with xtrace objects).
    """
    if status == NBX_OK:
        return
    if errors is None:
        from . import errors
    NumericalFault, PatternFault, ShapeMismatchError = (errors.NumericalFault, errors.PatternFault,
                                                        errors.ShapeMismatchError)
    msg = ctx.error()
    if status == NBX_ERR_NUMERICAL:
        if label == "simulate_image":  # which stage of the fused image faulted
            label = "nanobragg_spots" if ctx.lib.nbx_fault_stage(ctx.handle) == 0 else "add_background"
        cause = NumericalFault(first_bad)
        raise PatternFault(label, first_bad, cause) from cause
    if status == NBX_ERR_ARG:
        raise ShapeMismatchError(msg) if "dims" in msg or "buffer" in msg else ValueError(msg)
    raise NativeError(msg)
