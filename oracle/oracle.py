"""Python handle on the CPU oracle (TEST INFRASTRUCTURE ONLY).

Only tests/, __graft_entry__.smoke() and bench.py's CPU-baseline legs may
import this module; the product path never does.  It loads
oracle/_build/liboracle.so (built from oracle/nbx_oracle.c by oracle/Makefile,
rebuilt on demand) and evaluates a spot descriptor -- the same C struct the
GPU library consumes (include/nbx.h) -- with the reference's scalar FP64
formulation.  See the header of nbx_oracle.c for what it restates and how it
is pinned.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
LIB = HERE / "_build" / "liboracle.so"
SRC = [HERE / "nbx_oracle.c", HERE / "nbx_poisson_oracle.cpp", HERE / "Makefile",
       HERE.parent / "include" / "nbx.h", HERE.parent / "paper_2205_07976_b200" / "csrc" / "nbx_poisson.h"]

_lib = None


def build(force: bool = False) -> Path:
    stale = not LIB.exists() or any(p.stat().st_mtime > LIB.stat().st_mtime for p in SRC)
    if force or stale:
        res = subprocess.run(["make", "-C", str(HERE), "-B" if force else "-s"], capture_output=True, text=True)
        if res.returncode != 0:
            raise RuntimeError(f"oracle build failed:\n{res.stdout}\n{res.stderr}")
    return LIB


def load():
    global _lib
    if _lib is None:
        build()
        lib = C.CDLL(str(LIB))
        lib.oracle_spots.restype = C.c_int
        lib.oracle_spots.argtypes = [C.c_void_p, C.c_int, C.c_void_p, C.c_int, C.POINTER(C.c_int64)]
        lib.oracle_scale.restype = C.c_double
        lib.oracle_scale.argtypes = [C.c_void_p]
        lib.oracle_background.restype = C.c_int
        lib.oracle_background.argtypes = [C.c_void_p, C.c_int, C.c_void_p, C.POINTER(C.c_int64)]
        lib.oracle_poisson.restype = C.c_int
        lib.oracle_poisson.argtypes = [C.c_void_p, C.c_void_p, C.c_int64, C.c_int, C.c_uint64, C.c_uint64]
        _lib = lib
    return _lib


def threads() -> int:
    try:
        return len(os.sched_getaffinity(0))
    except AttributeError:  # pragma: no cover
        return os.cpu_count() or 1


def spots(desc, mode: str = "f64", nthreads: int | None = None, out: np.ndarray | None = None):
    """Evaluate a descriptor (paper_2205_07976_b200._native.Descriptor or its .c struct).

    mode: "f32" (the reference's stored image), "f64" (scale*acc before the
    cast -- the reference's 'oracle64'), "raw" (unscaled acc, added into
    ``out``).  Returns (image, first_bad).
    """
    lib = load()
    c = getattr(desc, "c", desc)
    n = sum(c.panels[i].slow_pixels * c.panels[i].fast_pixels for i in range(c.n_panels))
    code = {"f32": 0, "f64": 1, "raw": 3}[mode]
    if out is None:
        out = np.zeros(n, dtype=np.float32 if mode == "f32" else np.float64)
    bad = C.c_int64(-1)
    rc = lib.oracle_spots(C.addressof(c), code, out.ctypes.data, nthreads or threads(), C.byref(bad))
    if rc != 0:
        raise ValueError("oracle rejected the descriptor")
    return out, bad.value


def background(desc, mode: str = "f64"):
    """add_background restated (kernels.py:279-312); desc must carry the bg_* fields."""
    lib = load()
    c = getattr(desc, "c", desc)
    n = sum(c.panels[i].slow_pixels * c.panels[i].fast_pixels for i in range(c.n_panels))
    out = np.zeros(n, dtype=np.float32 if mode == "f32" else np.float64)
    bad = C.c_int64(-1)
    if lib.oracle_background(C.addressof(c), 0 if mode == "f32" else 1, out.ctypes.data, C.byref(bad)) != 0:
        raise ValueError("oracle rejected the background descriptor")
    return out, bad.value


def scale(desc) -> float:
    return load().oracle_scale(C.addressof(getattr(desc, "c", desc)))


def poisson(mean: np.ndarray, seed: int, image: int = 0) -> np.ndarray:
    """Host twin of the device Poisson sampler (same header, same bits)."""
    lib = load()
    mean = np.ascontiguousarray(mean)
    dtype = 1 if mean.dtype == np.float64 else 0
    if dtype == 0:
        mean = mean.astype(np.float32, copy=False)
    out = np.empty_like(mean)
    rc = lib.oracle_poisson(mean.ctypes.data, out.ctypes.data, mean.size, dtype, seed & (2**64 - 1),
                            image & (2**64 - 1))
    if rc != 0:
        raise ValueError("bad poisson arguments")
    return out
