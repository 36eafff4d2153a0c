"""Build the native library in-tree: paper_2205_07976_b200/_lib/libnbx.so.

nvcc cross-compiles for sm_100a only (no PTX fallback, no other arch).  The
library is the C ABI declared in include/nbx.h; Python binds it with ctypes
(_native.py).  Run ``python -m paper_2205_07976_b200.build`` or call
``build()``; it is also invoked by ``__graft_entry__.build()``.
"""
from __future__ import annotations

import os
import shutil
import subprocess
import sys
from pathlib import Path

PKG = Path(__file__).resolve().parent
ROOT = PKG.parent
CSRC = PKG / "csrc"
LIBDIR = PKG / "_lib"
LIB = LIBDIR / "libnbx.so"
SOURCES = ["nbx_kernels.cu", "nbx_reduce.cu", "nbx_runtime.cu"]
HEADERS = ["nbx_device.cuh", "nbx_kernels.cuh", "nbx_poisson.h"]

ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
NVCC_FLAGS = [
    "-O3", "-std=c++17", "-lineinfo", "--expt-relaxed-constexpr",
    "-Xcompiler", "-fPIC", "-Xcompiler", "-ffp-contract=off",
    "-Xptxas", "-v",
]


def nvcc() -> str:
    for cand in (os.environ.get("NVCC"), "/usr/local/cuda/bin/nvcc", shutil.which("nvcc")):
        if cand and Path(cand).exists():
            return cand
    raise RuntimeError("nvcc not found; the native library cannot be built")


def _stale() -> bool:
    if not LIB.exists():
        return True
    t = LIB.stat().st_mtime
    deps = [CSRC / s for s in SOURCES + HEADERS] + [ROOT / "include" / "nbx.h"]
    return any(p.stat().st_mtime > t for p in deps)


def build(force: bool = False, verbose: bool = False, extra_flags: list[str] | None = None,
          out: Path | None = None) -> Path:
    """Compile the sources and link libnbx.so; returns its path.

    ``extra_flags``/``out`` build an experimental variant (e.g. -DNBX_MIN_BLOCKS_F32=4) elsewhere.
    """
    lib = Path(out) if out else LIB
    if not force and out is None and not _stale():
        return LIB
    lib.parent.mkdir(parents=True, exist_ok=True)
    LIBDIR.mkdir(exist_ok=True)
    from concurrent.futures import ThreadPoolExecutor

    def compile_one(src):
        obj = lib.parent / (lib.stem + "_" + Path(src).stem + ".o")
        cmd = [nvcc(), *ARCH, *NVCC_FLAGS, *(extra_flags or []), "-I", str(ROOT / "include"), "-c",
               str(CSRC / src), "-o", str(obj)]
        return src, obj, subprocess.run(cmd, capture_output=True, text=True)

    objs = []
    logs = []
    with ThreadPoolExecutor(max_workers=len(SOURCES)) as pool:  # the translation units compile in parallel
        for src, obj, res in pool.map(compile_one, SOURCES):
            logs.append(res.stderr)
            if res.returncode != 0:
                raise RuntimeError(f"nvcc failed on {src}:\n{res.stderr}")
            objs.append(str(obj))
    tmp = lib.with_suffix(".so.tmp")
    cmd = [nvcc(), *ARCH, "-shared", "-o", str(tmp), *objs, "-lcudart"]
    res = subprocess.run(cmd, capture_output=True, text=True)
    if res.returncode != 0:
        raise RuntimeError(f"link failed:\n{res.stderr}")
    os.replace(tmp, lib)
    (lib.parent / (lib.stem + "_ptxas.log" if out else "ptxas.log")).write_text("\n".join(logs))
    if verbose:
        sys.stdout.write("\n".join(logs))
    return lib


if __name__ == "__main__":
    path = build(force="--force" in sys.argv, verbose="-v" in sys.argv)
    print(path)
