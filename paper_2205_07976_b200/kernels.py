"""The spot kernel behind the reference's plugin API.

Drop-in for the reference's spot path (/root/reference/pkg/src/xtrace/kernels.py):

    nanobragg_spots(ctx: SpotsContext, out: PixelBuffer, executor=None) -> None

Same arguments, same in-place write into ``out.data``, same errors
(ShapeMismatchError for dims/precision, PatternFault(label, pixel,
NumericalFault(pixel)) for the lowest non-finite pixel).  The pixels are
computed by the hand-written sm_100a kernel in csrc/ through the C ABI
(include/nbx.h); ``executor`` is accepted for signature compatibility (the
call logs no timing record of its own, as the reference's body does not:
``kernel_timer`` around it does).  With the reference's own objects as inputs
the errors raised are the reference's classes (``xtrace.errors``).  There is
no CPU fallback.

Extensions (all default to the reference behaviour):
  SpotsContext.compute  "fp64" (default; the reference's FP64 arithmetic) or
                        "fp32" (FP64 geometry/phase, FP32 sin/ratio; 1e-4 parity)
  SpotsContext.shape    "sincg" (reference) | "gauss" | "round" | "tophat"
  SpotsContext.phi      PhiScan (spindle steps)
  panel may be a Detector (several panels, one launch)
  out.precision "f64"   FP64 store (the reference only accepts f32)
"""
from __future__ import annotations

import math
import time
import weakref
from dataclasses import dataclass

import numpy as np

from . import _native as N
from . import errors as _errors
from .errors import ShapeMismatchError
from .model import BeamSpectrum, CrystalModel, Detector, DetectorPanel, PhiScan

__all__ = [
    "R_E_SQR",
    "KERNEL_GRAIN",
    "PixelBuffer",
    "SpotsContext",
    "SpotsPlan",
    "sincg",
    "lattice_transform",
    "nanobragg_spots",
    "add_array",
    "add_background",
    "simulate_image",
    "add_noise",
    "poisson_host",
    "describe",
]

R_E_SQR = 7.94079248e-30  # classical electron radius squared, m^2 (kernels.py:44)
KERNEL_GRAIN = 4096        # kept for API compatibility; the GPU grid does not use it
_SINC_LIMIT = 1e-12
_DTYPES = {"f32": np.float32, "f64": np.float64}


class PixelBuffer:
    """Flat row-major image (slow outermost) of fixed precision (kernels.py:57-97)."""

    __slots__ = ("data", "dims", "precision")

    def __init__(self, dims: tuple[int, int], precision: str = "f32", data=None):
        if precision not in _DTYPES:
            raise ValueError("precision must be 'f32' or 'f64'")
        slow, fast = int(dims[0]), int(dims[1])
        if slow < 1 or fast < 1:
            raise ValueError("buffer dims must be positive")
        dtype = _DTYPES[precision]
        if data is None:
            data = np.zeros(slow * fast, dtype=dtype)
        else:
            data = np.asarray(data, dtype=dtype).reshape(-1)
            if data.size != slow * fast:
                raise ShapeMismatchError(f"buffer length {data.size} != {slow}x{fast}")
        self.data = data
        self.dims = (slow, fast)
        self.precision = precision

    @classmethod
    def zeros(cls, dims, precision="f32"):
        return cls(dims, precision)

    @property
    def n_pixels(self) -> int:
        return self.data.size

    def as_image(self) -> np.ndarray:
        return self.data.reshape(self.dims)

    def copy(self) -> "PixelBuffer":
        return PixelBuffer(self.dims, self.precision, self.data.copy())

    def __repr__(self):
        return f"PixelBuffer({self.dims}, {self.precision})"


@dataclass(frozen=True)
class SpotsContext:
    """Read-only inputs of the spot kernel (kernels.py:100-112) plus extensions."""

    crystal: CrystalModel
    panel: DetectorPanel | Detector
    spectrum: BeamSpectrum
    oversample: int = 1
    r_e_sqr: float = R_E_SQR
    compute: str = "fp64"
    shape: str = "sincg"
    phi: PhiScan | None = None

    def __post_init__(self):
        if self.oversample < 1:
            raise ValueError("oversample must be >= 1")
        if self.compute not in N.COMPUTE:
            raise ValueError(f"compute must be one of {sorted(N.COMPUTE)}")
        if self.shape not in N.SHAPES:
            raise ValueError(f"shape must be one of {sorted(N.SHAPES)}")


def sincg(x: float, n: int) -> float:
    """sin(n x)/sin(x) with the analytic limit near sin x = 0 (kernels.py:115-120).

    Host-side scalar helper (used for golden values and the facade); the
    image path evaluates the same function on the GPU.
    """
    sx = math.sin(x)
    if abs(sx) < _SINC_LIMIT:
        return n * math.cos(n * x) / math.cos(x)
    return math.sin(n * x) / sx


def lattice_transform(crystal: CrystalModel, h: float, k: float, l: float) -> float:
    """Grating amplitude at fractional Miller coordinates (kernels.py:123-131)."""
    na, nb, nc = crystal.n_cells
    return sincg(math.pi * h, na) * sincg(math.pi * k, nb) * sincg(math.pi * l, nc)


def _panels_of(panel) -> tuple:
    return panel.panels if isinstance(panel, (Detector, DetectorPanel)) else (panel,)


_XTABLE_CACHE: "weakref.WeakKeyDictionary" = weakref.WeakKeyDictionary()


def _table_arrays(table) -> tuple[np.ndarray, np.ndarray]:
    if hasattr(table, "arrays"):
        return table.arrays()
    # The reference's StructureFactorTable (model.py:227-285) keeps its entries packed and
    # sorted for its own vectorised lookup (_packed_keys = (h+2^20)<<42 | (k+2^20)<<21 |
    # (l+2^20), model.py:249-259): unpack those (about 1 ms for 178k entries instead of ~57 ms
    # walking the dict) and remember the result per table object.
    keys, vals = getattr(table, "_packed_keys", None), getattr(table, "_packed_vals", None)
    if isinstance(keys, np.ndarray) and isinstance(vals, np.ndarray) and keys.shape == vals.shape:
        try:
            hit = _XTABLE_CACHE.get(table)
        except TypeError:  # not weak-referenceable
            hit = None
        if hit is not None and hit[0] is keys:
            return hit[1], hit[2]
        b = np.int64(1 << 20)
        k = keys.astype(np.int64)
        hkl = np.stack([(k >> 42) - b, ((k >> 21) & 0x1FFFFF) - b, (k & 0x1FFFFF) - b], axis=1).astype(np.int32)
        amp = np.ascontiguousarray(vals, dtype=np.float64)
        try:
            _XTABLE_CACHE[table] = (keys, hkl, amp)
        except TypeError:
            pass
        return hkl, amp
    # any other duck-typed table: a dict of entries
    n = len(table.entries)
    hkl = np.array(list(table.entries.keys()), dtype=np.int32).reshape(n, 3)
    amp = np.array(list(table.entries.values()), dtype=np.float64).reshape(n)
    return hkl, amp


def describe(ctx, *, src_begin: int = 0, src_end: int = 0, norm: float = 0.0, background=None,
             thickness_factor: float = 1.0) -> N.Descriptor:
    """Flatten a SpotsContext into the C descriptor (what the kernel reads).

    Accepts this package's SpotsContext or the reference's own (duck typing:
    crystal/panel/spectrum/oversample/r_e_sqr with the reference's fields), so
    ``nanobragg_spots(xtrace_ctx, xtrace_pixelbuffer)`` works unchanged.
    """
    crystal, spectrum = ctx.crystal, ctx.spectrum
    hkl, amp = _table_arrays(crystal.sf_table)
    phi = getattr(ctx, "phi", None)
    bases = crystal.rotated_real_bases(phi) if phi is not None else crystal.rotated_real_bases()
    return N.Descriptor(
        panels=_panels_of(ctx.panel),
        oversample=ctx.oversample,
        beam_direction=spectrum.beam_direction,
        polarization_on=spectrum.polarization_on,
        wavelengths=spectrum.wavelengths,
        weights=spectrum.weights,
        fluence=spectrum.fluence,
        r_e_sqr=ctx.r_e_sqr,
        bases=bases,
        n_cells=crystal.n_cells,
        hkl=hkl,
        amplitudes=amp,
        default_f=crystal.sf_table.default_f,
        shape=N.SHAPES[getattr(ctx, "shape", "sincg")],
        norm=norm,
        src_begin=src_begin,
        src_end=src_end,
        background=background,
        thickness_factor=thickness_factor,
    )


def _dims_of(panel) -> tuple[int, int]:
    return panel.dims


def _check_out(out: PixelBuffer, panel, errors=None):
    # kernels.py:204-208 (f64 is accepted here as an extension)
    err = (errors or _errors).ShapeMismatchError
    if out.dims != _dims_of(panel):
        raise err(f"buffer dims {out.dims} != panel dims {_dims_of(panel)}")
    if out.precision not in _DTYPES:
        raise err(f"unsupported buffer precision {out.precision}")
    if not (out.data.flags.c_contiguous and out.data.flags.writeable):
        raise err("output buffer must be a contiguous writeable array")


def nanobragg_spots(ctx: SpotsContext, out: PixelBuffer, executor=None) -> None:
    """Simulate the Bragg-spot image into ``out`` on the GPU (kernels.py:219-276).

    out[p] = r_e^2 * fluence / (sum(w) * n_domains * oversample^2)
             * sum_{sub, domain, source} w * Omega*pol(sub) * (F_cell * F_latt)^2
    """
    errors = _errors.hierarchy_for(ctx, out)  # xtrace objects in -> xtrace.errors classes out
    _check_out(out, ctx.panel, errors)
    desc = describe(ctx)
    cx = N.context()
    mode = N.OUT_F32 if out.precision == "f32" else N.OUT_F64
    bad = N.C.c_int64(-1)
    compute = N.COMPUTE[getattr(ctx, "compute", "fp64")]
    with cx.lock:
        status = cx.lib.nbx_spots(cx.handle, N.C.byref(desc.c), compute, mode,
                                  out.data.ctypes.data, 0, N.C.byref(bad))
        N.check(cx, status, bad.value, errors=errors)
    # no timing record here: like the reference body (parallel_for_blocks, execution.py:207-224),
    # the call itself logs nothing; callers time it with kernel_timer (execution.py:350-356)


class SpotsPlan:
    """Inputs of one SpotsContext resident in HBM, runnable many times.

    ``run(out_ptr, on_device=True)`` writes straight into device memory (e.g.
    a torch tensor's ``data_ptr()``); ``kernel_ms`` is the CUDA-event time of
    the last spot kernel.
    """

    def __init__(self, ctx: SpotsContext, *, device: int | None = None, src_begin: int = 0,
                 src_end: int = 0, norm: float = 0.0):
        self.cx = N.context(device)
        self.desc = describe(ctx, src_begin=src_begin, src_end=src_end, norm=norm)
        with self.cx.lock:
            self.handle = self.cx.lib.nbx_plan_create(self.cx.handle, N.C.byref(self.desc.c),
                                                      N.COMPUTE[ctx.compute])
            if not self.handle:
                N.check(self.cx, N.NBX_ERR_ARG if "cuda" not in self.cx.error().lower() else N.NBX_ERR_CUDA)
            info = N.PlanInfo()
            self.cx.lib.nbx_plan_info(self.handle, N.C.byref(info))
        self.info = info
        self.dims = _dims_of(ctx.panel)

    @property
    def steps(self) -> int:
        return int(self.info.steps)

    @property
    def n_pixels(self) -> int:
        return int(self.info.n_pixels)

    @property
    def scale(self) -> float:
        return float(self.info.scale)

    def run(self, out, *, mode: int = N.OUT_F32, on_device: bool = False) -> None:
        """Run into ``out``: a PixelBuffer / NumPy array (host) or a device pointer (int)."""
        if isinstance(out, PixelBuffer):
            out = out.data
        if isinstance(out, np.ndarray):
            want = np.float32 if mode == N.OUT_F32 else np.float64
            if out.dtype != want or out.size != self.n_pixels or not out.flags.c_contiguous:
                raise ShapeMismatchError("output array does not match the plan")
            addr, dev = out.ctypes.data, 0
        else:
            addr, dev = int(out), 1 if on_device else 0
        bad = N.C.c_int64(-1)
        with self.cx.lock:
            status = self.cx.lib.nbx_plan_run(self.handle, mode, addr, dev, N.C.byref(bad))
            N.check(self.cx, status, bad.value)

    @property
    def kernel_ms(self) -> float:
        return float(self.cx.lib.nbx_plan_last_kernel_ms(self.handle))

    def close(self):
        if getattr(self, "handle", None):
            with self.cx.lock:
                self.cx.lib.nbx_plan_destroy(self.handle)
                self.handle = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def _bg_descriptor(profile, panel, spectrum, thickness_factor: float) -> N.Descriptor:
    """Descriptor carrying only what the background kernel reads."""
    return N.Descriptor(
        panels=_panels_of(panel), oversample=1, beam_direction=spectrum.beam_direction,
        polarization_on=spectrum.polarization_on, wavelengths=spectrum.wavelengths, weights=spectrum.weights,
        fluence=spectrum.fluence, r_e_sqr=R_E_SQR, bases=np.eye(3)[None], n_cells=(1, 1, 1),
        hkl=np.zeros((0, 3), np.int32), amplitudes=np.zeros(0), default_f=0.0, background=profile,
        thickness_factor=thickness_factor)


def add_background(profile, panel, spectrum, thickness_factor: float, out: PixelBuffer, executor=None) -> None:
    """Diffuse (air/water) background into ``out`` on the GPU (kernels.py:279-312).

    out[p] = r_e^2 fluence thickness_factor / sum(w) * sum_w w f_bg(sin(theta)/lambda_w)^2 * Omega*pol,
    at pixel centres.  f32 store (the reference) or f64 (extension).
    """
    errors = _errors.hierarchy_for(profile, panel, spectrum, out)
    _check_out(out, panel, errors)
    desc = _bg_descriptor(profile, panel, spectrum, thickness_factor)
    cx = N.context()
    bad = N.C.c_int64(-1)
    mode = N.OUT_F32 if out.precision == "f32" else N.OUT_F64
    with cx.lock:
        status = cx.lib.nbx_background(cx.handle, N.C.byref(desc.c), mode, out.data.ctypes.data, 0,
                                       N.C.byref(bad))
        N.check(cx, status, bad.value, label="add_background", errors=errors)
    # no timing record (the reference body logs nothing; kernel_timer does)


def simulate_image(ctx, background=None, thickness_factor: float = 1.0, out: PixelBuffer | None = None,
                   executor=None) -> PixelBuffer:
    """One image's 64-bit accumulator, spots + background fused in ONE launch (scheduler.py:156-183).

    Equals the reference pipeline bit for bit in structure: f64(f32(spots)) then
    + f64(f32(background)) (add_array, kernels.py:315-331), with the spot and
    background stages evaluated by the same kernel and no 32-bit staging
    buffers in HBM.  ``background=None`` skips the background stage.

    Also accepts the reference's own signature ``simulate_image(config, image_seed,
    executor=None)`` with a ``SimulationConfig``-like ``config`` (``crystal_for_seed``,
    ``panel``, ``spectrum``, ``oversample``, ``background``, ``thickness_factor``;
    io.py:122-157), FP64 path as in the reference.  The executor then receives one
    ("simulate_image", ms) record for the fused launch.
    """
    if hasattr(ctx, "crystal_for_seed"):  # scheduler.py:156-183 signature
        config, image_seed = ctx, background
        if image_seed is None or isinstance(image_seed, bool):
            raise TypeError("simulate_image(config, image_seed, executor=None) needs an integer image_seed")
        if executor is None and not isinstance(thickness_factor, (int, float)):
            executor = thickness_factor  # positional executor, the reference's third argument
        sctx = SpotsContext(config.crystal_for_seed(int(image_seed)), config.panel, config.spectrum,
                            int(getattr(config, "oversample", 1)))
        return simulate_image(sctx, background=getattr(config, "background", None),
                              thickness_factor=float(getattr(config, "thickness_factor", 1.0)), out=out,
                              executor=executor)
    dims = ctx.panel.dims
    if out is None:
        out = PixelBuffer.zeros(dims, "f64")
    _check_out(out, ctx.panel)
    if out.precision != "f64":
        raise ShapeMismatchError("simulate_image accumulates into an f64 buffer")
    t0 = time.perf_counter()
    desc = describe(ctx, background=background, thickness_factor=thickness_factor)
    cx = N.context()
    bad = N.C.c_int64(-1)
    with cx.lock:
        status = cx.lib.nbx_spots(cx.handle, N.C.byref(desc.c), N.COMPUTE[getattr(ctx, "compute", "fp64")],
                                  N.OUT_IMAGE_F64, out.data.ctypes.data, 0, N.C.byref(bad))
        N.check(cx, status, bad.value, label="simulate_image")
    if executor is not None and hasattr(executor, "timing_log"):
        from .execution import TimingRecord

        executor.timing_log.append(TimingRecord("simulate_image", (time.perf_counter() - t0) * 1e3))
    return out


def add_array(lhs: PixelBuffer, rhs: PixelBuffer, executor=None) -> None:
    """lhs[j] += float64(rhs[j]) on the GPU (kernels.py:315-331)."""
    if lhs.dims != rhs.dims:
        raise ShapeMismatchError(f"dims {lhs.dims} != {rhs.dims}")
    if lhs.precision != "f64" or rhs.precision != "f32":
        raise ShapeMismatchError("add_array expects f64 lhs and f32 rhs")
    cx = N.context()
    rhs_data = np.ascontiguousarray(rhs.data)
    with cx.lock:
        status = cx.lib.nbx_add_array(cx.handle, lhs.data.ctypes.data, rhs_data.ctypes.data, lhs.n_pixels, 0)
        N.check(cx, status, label="add_array")


def add_noise(buf: PixelBuffer, seed: int, image: int = 0) -> PixelBuffer:
    """Poisson photon counts drawn around ``buf``, on the GPU.

    Counter-based Philox keyed by (seed, image), counter = pixel, so the draw
    is reproducible and bit-identical to ``poisson_host``.
    """
    cx = N.context()
    out = PixelBuffer(buf.dims, buf.precision)
    dtype = 0 if buf.precision == "f32" else 1
    src = np.ascontiguousarray(buf.data)
    with cx.lock:
        status = cx.lib.nbx_add_noise(cx.handle, src.ctypes.data, out.data.ctypes.data, buf.n_pixels, dtype,
                                      int(seed) & (2**64 - 1), int(image) & (2**64 - 1), 0)
        N.check(cx, status, label="add_noise")
    return out


def poisson_host(buf: PixelBuffer, seed: int, image: int = 0) -> PixelBuffer:
    """CPU twin of add_noise (same header, same bits) -- the noise oracle."""
    lib = N.load()
    out = PixelBuffer(buf.dims, buf.precision)
    dtype = 0 if buf.precision == "f32" else 1
    src = np.ascontiguousarray(buf.data)
    status = lib.nbx_poisson_host(src.ctypes.data, out.data.ctypes.data, buf.n_pixels, dtype,
                                  int(seed) & (2**64 - 1), int(image) & (2**64 - 1))
    if status != N.NBX_OK:
        raise ValueError("invalid poisson_host arguments")
    return out


def __getattr__(name):
    # image_stats / image_histogram live in xtrace.kernels (kernels.py:334-430); here they are
    # implemented next to the image I/O (io.py) and re-exported lazily (io imports this module)
    if name in ("image_stats", "image_histogram", "ImageStats", "HistogramResult"):
        from . import io

        return getattr(io, name)
    raise AttributeError(f"module {__name__!r} has no attribute {name!r}")

