"""A plain-C host program against include/nbx.h + libnbx.so (examples/nbx_c1_demo.c), no
Python on the GPU path: it builds the C1 acceptance toy's descriptor itself, renders it with
nbx_spots on both compute paths and re-runs it through a resident plan.  Its images must equal
the Python drop-in API's (which reaches the same library through ctypes) bit for bit."""
import subprocess
from pathlib import Path

import numpy as np
import pytest

from paper_2205_07976_b200 import PixelBuffer, nanobragg_spots, synthetic

ROOT = Path(__file__).resolve().parents[1]
LIBDIR = ROOT / "paper_2205_07976_b200" / "_lib"
pytestmark = pytest.mark.gpu


def test_c_host_program_matches_python_api(gpu, tmp_path):
    exe = tmp_path / "nbx_c1_demo"
    subprocess.run(["cc", "-O2", "-Wall", "-Wextra", "-Werror", "-I", str(ROOT / "include"),
                    str(ROOT / "examples" / "nbx_c1_demo.c"), "-L", str(LIBDIR), "-lnbx",
                    f"-Wl,-rpath,{LIBDIR}", "-lm", "-o", str(exe)], check=True)
    res = subprocess.run([str(exe), str(tmp_path / "c1")], capture_output=True, text=True, timeout=300)
    assert res.returncode == 0, res.stderr
    assert res.stdout.count("plan re-run mismatches 0") == 2, res.stdout
    for compute in ("fp64", "fp32"):
        got = np.fromfile(tmp_path / f"c1.{compute}.f32", dtype=np.float32)
        want = PixelBuffer.zeros((256, 256), "f32")
        nanobragg_spots(synthetic.c1_context(compute), want)
        assert np.array_equal(got, want.data), compute
