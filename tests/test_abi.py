"""The C-ABI library builds, loads and exports exactly what include/nbx.h declares (CPU-only)."""
import ctypes as C
import re
from pathlib import Path

import numpy as np
import pytest

from paper_2205_07976_b200 import _native, build

ROOT = Path(__file__).resolve().parents[1]


@pytest.fixture(scope="module")
def lib():
    build.build()
    return _native.load()


def header_functions():
    text = (ROOT / "include" / "nbx.h").read_text()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return set(re.findall(r"\b(nbx_\w+)\s*\(", text))


def test_header_matches_binding_table():
    assert header_functions() == set(_native.EXPORTS)


def test_every_symbol_exported(lib):
    for name in _native.EXPORTS:
        assert hasattr(lib, name), name


def test_library_is_sm100a_only():
    out = __import__("subprocess").run(["cuobjdump", "--list-elf", str(_native.LIB_PATH)],
                                       capture_output=True, text=True).stdout
    assert "sm_100a" in out
    assert not re.search(r"sm_(?!100a)\d+", out)


def test_version(lib):
    assert lib.nbx_version() == 10000


def test_no_gpu_fails_loudly_here(lib):
    import torch

    if torch.cuda.is_available():
        pytest.skip("GPU present")
    assert not lib.nbx_ctx_create(0)
    assert b"device" in lib.nbx_last_error(None)
    with pytest.raises(_native.NativeError):
        _native.Context(0)
    _native._lib = None  # first use through context() must not deadlock on the loader lock
    with pytest.raises(_native.NativeError):
        _native.context(0)


def test_output_pixels_is_host_only(lib):
    from paper_2205_07976_b200 import synthetic

    desc = __import__("paper_2205_07976_b200").describe(synthetic.c1_context())
    assert lib.nbx_output_pixels(C.byref(desc.c)) == 256 * 256
    desc.c.panels[0].slow_pixels = 0
    assert lib.nbx_output_pixels(C.byref(desc.c)) == -1


def test_struct_layout_matches_header():
    # offsets the C compiler gives nbx_spots_desc, checked via a tiny C probe
    import subprocess
    import tempfile

    probe = r'''
#include <stdio.h>
#include <stddef.h>
#include "nbx.h"
int main(){printf("%zu %zu %zu %zu %zu %zu %zu\n", sizeof(nbx_panel), sizeof(nbx_spots_desc),
 offsetof(nbx_spots_desc, bases), offsetof(nbx_spots_desc, default_f), offsetof(nbx_spots_desc, src_end),
 sizeof(nbx_plan_info_t), offsetof(nbx_panel, attenuation_length));return 0;}
'''
    with tempfile.TemporaryDirectory() as d:
        src = Path(d) / "p.c"
        src.write_text(probe)
        exe = Path(d) / "p"
        subprocess.run(["gcc", "-I", str(ROOT / "include"), str(src), "-o", str(exe)], check=True)
        got = [int(x) for x in subprocess.run([str(exe)], capture_output=True, text=True).stdout.split()]
    want = [C.sizeof(_native.Panel), C.sizeof(_native.SpotsDesc), _native.SpotsDesc.bases.offset,
            _native.SpotsDesc.default_f.offset, _native.SpotsDesc.src_end.offset, C.sizeof(_native.PlanInfo),
            _native.Panel.attenuation_length.offset]
    assert got == want


def test_host_poisson_twin_matches_oracle_build(lib):
    """nbx_poisson_host (product .so, nvcc host build) == oracle build (g++): same header, same bits."""
    from oracle import oracle

    rng = np.random.default_rng(5)
    mean = np.concatenate([rng.uniform(0, 15, 4000), rng.uniform(15, 1e5, 4000), [0.0, -1.0, 1e9]])
    out = np.empty_like(mean)
    assert lib.nbx_poisson_host(mean.ctypes.data, out.ctypes.data, mean.size, 1, 77, 3) == 0
    assert np.array_equal(out, oracle.poisson(mean, 77, 3))


def test_crc32_matches_zlib(lib):
    import zlib

    for n in (0, 1, 7, 8, 9, 4096, 100003):
        b = np.random.default_rng(n).integers(0, 256, n, dtype=np.uint8)
        assert lib.nbx_crc32(0, b.ctypes.data, n) == zlib.crc32(b.tobytes())


def test_struct_mirrors_match_the_library(lib):
    """The ctypes mirrors (_native.py) have the sizes the library was compiled with."""
    lib.nbx_struct_size.restype = C.c_int64
    assert lib.nbx_struct_size(0) == C.sizeof(_native.Panel)
    assert lib.nbx_struct_size(1) == C.sizeof(_native.SpotsDesc)
    assert lib.nbx_struct_size(2) == C.sizeof(_native.PlanInfo)
    assert lib.nbx_struct_size(7) == 0


def test_integration_doc_binding_matches_the_library(lib):
    """The self-contained ctypes binding shown in INTEGRATION.md section 2 is ABI-correct."""
    text = (ROOT / "INTEGRATION.md").read_text()
    block = text.split("## 2. Raw C ABI", 1)[1].split("```python", 1)[1].split("```", 1)[0]
    structs = block.split("lib.nbx_struct_size.restype", 1)[0]  # imports + the two Structure classes
    ns = {}
    exec(compile(structs.replace('lib = C.CDLL("/path/to/paper_2205_07976_b200/_lib/libnbx.so")', ""),
                 "INTEGRATION.md", "exec"), ns)
    lib.nbx_struct_size.restype = C.c_int64
    assert lib.nbx_struct_size(0) == C.sizeof(ns["Panel"])
    assert lib.nbx_struct_size(1) == C.sizeof(ns["Desc"])
    assert [f[0] for f in ns["Desc"]._fields_] == [f[0] for f in _native.SpotsDesc._fields_]


def test_default_device_follows_nbx_device_then_local_rank(monkeypatch):
    """The default context's device: NBX_DEVICE wins; under torchrun LOCAL_RANK wrapped onto the
    visible devices (0 here: no GPU in this container, nbx_device_count() == 0)."""
    monkeypatch.setenv("NBX_DEVICE", "3")
    assert _native.default_device() == 3
    monkeypatch.delenv("NBX_DEVICE")
    monkeypatch.setenv("LOCAL_RANK", "5")
    n = _native.load().nbx_device_count()
    assert n >= 0
    torch = __import__("sys").modules.get("torch")
    if torch is None or not torch.cuda.is_initialized():
        assert _native.default_device() == (5 % n if n else 0)


def test_missing_native_library_fails_loudly(tmp_path):
    """No CPU fallback: with the library absent the drop-in call raises NativeError (a fresh
    interpreter with NBX_LIB pointing at a missing file)."""
    import subprocess
    import sys

    code = ("import sys; sys.path.insert(0, %r)\n"
            "from paper_2205_07976_b200 import PixelBuffer, nanobragg_spots, synthetic\n"
            "from paper_2205_07976_b200.errors import NativeError\n"
            "ctx = synthetic.c1_context()\n"
            "try:\n"
            "    nanobragg_spots(ctx, PixelBuffer.zeros(ctx.panel.dims))\n"
            "except NativeError as e:\n"
            "    print('NativeError', e)\n" % str(Path(__file__).resolve().parents[1]))
    env = dict(__import__("os").environ, NBX_LIB=str(tmp_path / "absent.so"))
    res = subprocess.run([sys.executable, "-c", code], capture_output=True, text=True, env=env, timeout=300)
    assert res.returncode == 0, res.stderr
    assert res.stdout.startswith("NativeError native library missing"), res.stdout
