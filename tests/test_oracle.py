"""The CPU oracle (oracle/) is pinned against the reference's own outputs and known answers (CPU-only)."""
import math

import numpy as np
import pytest

import parity
from oracle import oracle
from paper_2205_07976_b200 import (
    CrystalModel,
    MosaicDomainSet,
    Orientation,
    StructureFactorTable,
    UnitCell,
    describe,
    lattice_transform,
    sincg,
)

CASES = ["thomson", "scalar_match", "triclinic_pol_2wl", "pipeline_spots", "c1_toy", "tilted", "ls49_centre",
         "ls49_edge"]


def crystal(n_cells=(5, 5, 5)):
    return CrystalModel(UnitCell(100, 100, 100, 90, 90, 90), Orientation(), n_cells,
                        MosaicDomainSet(np.eye(3)[None]), StructureFactorTable({}, 100.0))


# known-answer values frozen in the reference tests (test_kernels.py:40,64-90)
def test_sincg_golden():
    assert sincg(0.0, 5) == 5.0
    assert sincg(math.pi / 2, 2) == pytest.approx(0.0, abs=1e-15)
    assert sincg(0.3, 4) == pytest.approx(3.153892914792541, rel=1e-15)


def test_lattice_transform_golden():
    assert abs(lattice_transform(crystal((5, 5, 5)), 2.0, -3.0, 1.0)) == 125.0
    assert abs(lattice_transform(crystal((3, 4, 7)), 1.0, 0.0, -2.0)) == 84.0
    assert abs(lattice_transform(crystal((5, 1, 1)), 0.2, 0.0, 0.0)) < 1e-9
    assert lattice_transform(crystal((4, 1, 1)), 0.3, 0.0, 0.0) == pytest.approx(-0.7265425280053609, rel=1e-14)


@pytest.mark.parametrize("name", CASES)
def test_oracle_matches_reference_fixture(name):
    case = parity.load(name)
    desc = describe(parity.context(case))
    f64, bad = oracle.spots(desc, "f64")
    assert bad == -1
    ref = case["ref_f64"]
    m = parity.metrics(f64, ref, (int(case["panel"][0]), int(case["panel"][1])))
    assert m["total"] < 1e-12, m
    assert m["spot"] < 1e-11, m
    assert m["pix_abs_over_max"] < 1e-11, m
    f32, _ = oracle.spots(desc, "f32")
    same = np.mean(f32 == case["ref_f32"])
    assert same > 0.99, same
    ulp = np.abs(f32.astype(np.float64) - case["ref_f32"]) / np.maximum(np.abs(case["ref_f32"]), 1e-300)
    assert ulp.max() <= 2.0 ** -23


def test_oracle_scaling_laws_exact():
    case = parity.load("scalar_match")
    base = describe(parity.context(case))
    img, _ = oracle.spots(base, "f32")
    desc2 = describe(parity.context(case))
    desc2.c.fluence = base.c.fluence * 2
    img2, _ = oracle.spots(desc2, "f32")
    assert np.array_equal(img2, 2 * img)


def test_oracle_channel_shards_sum_to_whole():
    case = parity.load("pipeline_spots")
    whole = describe(parity.context(case))
    raw_whole, _ = oracle.spots(whole, "raw")
    acc = np.zeros_like(raw_whole)
    for lo, hi in ((0, 1), (1, 2)):
        part = describe(parity.context(case), src_begin=lo, src_end=hi)
        oracle.spots(part, "raw", out=acc)
    np.testing.assert_allclose(acc, raw_whole, rtol=1e-15, atol=0)


def test_oracle_threads_bitwise_invariant():
    case = parity.load("c1_toy")
    desc = describe(parity.context(case))
    a, _ = oracle.spots(desc, "f64", nthreads=1)
    b, _ = oracle.spots(desc, "f64", nthreads=7)
    assert np.array_equal(a, b)


def test_oracle_fault_pixel():
    case = parity.load("thomson")
    desc = describe(parity.context(case))
    desc.c.fluence = 1e300
    desc.c.default_f = 1e30
    _, bad = oracle.spots(desc, "f32")
    assert bad == 0


@pytest.mark.parametrize("name", ["bg_flat", "bg_scalar", "bg_water_80"])
def test_oracle_background_matches_reference_fixture(name):
    from paper_2205_07976_b200.kernels import _bg_descriptor

    case = parity.load(name)
    desc = _bg_descriptor(*parity.bg_inputs(case))
    got, bad = oracle.background(desc, "f64")
    assert bad == -1
    np.testing.assert_allclose(got, case["ref_bg_f64"], rtol=1e-13, atol=0)
    f32, _ = oracle.background(desc, "f32")
    assert np.mean(f32 == case["ref_bg_f32"]) > 0.99


def test_oracle_pipeline_matches_reference_fixture():
    from paper_2205_07976_b200.kernels import _bg_descriptor

    case = parity.load("pipeline_full")
    spots, _ = oracle.spots(describe(parity.context(case)), "f32")
    bg, _ = oracle.background(_bg_descriptor(*parity.bg_inputs(case)), "f32")
    acc = spots.astype(np.float64) + bg.astype(np.float64)
    np.testing.assert_allclose(acc, case["ref_image"], rtol=1e-7, atol=0)


def _stats_values(n, precision):
    rng = np.random.default_rng(n)  # tools/make_golden.py:stats_values
    return np.exp(rng.normal(0.0, 8.0, n)).astype(np.float32 if precision == "f32" else np.float64)


def reference_stats_total(values):
    """The reference image_stats total restated with NumPy (kernels.py:346-371, execution.py:227-260)."""
    blocks = [float(np.sum(values[i:i + 8192], dtype=np.float64)) for i in range(0, values.size, 8192)]

    def span(lo, hi):
        if hi - lo == 1:
            return blocks[lo]
        mid = lo + (1 << ((hi - lo - 1).bit_length() - 1))
        return span(lo, mid) + span(mid, hi)

    return span(0, len(blocks))


def test_stats_restatement_is_the_reference():
    """tests/golden/stats.npz holds xtrace.kernels.image_stats outputs (run by tools/make_golden.py);
    the NumPy restatement the GPU test compares against reproduces them bit for bit."""
    z = np.load(parity.GOLDEN / "stats.npz")
    for n, prec, ref in zip(z["n"], z["precision"], z["ref_stats"]):
        v = _stats_values(int(n), str(prec))
        total = reference_stats_total(v)
        assert total == ref[3]
        assert total / n == ref[2]
        assert float(v.min()) == ref[0] and float(v.max()) == ref[1]


def test_background_division_identity_is_correctly_rounded():
    """The background kernel's sin(theta)/lambda (nbx_kernels.cu:div_exact): q0 = RN(x inv),
    r = x - q0 lambda (exact, FMA), RN(q0 + r inv) with inv = RN(1/lambda) equals the IEEE
    quotient NumPy computes.  Checked with exact rational arithmetic on seeded samples over the
    range the kernel sees (x = sin(theta) in [0, 1], lambda in Angstrom)."""
    import random
    from fractions import Fraction

    rng = random.Random(7)
    for i in range(20000):
        x = rng.random() if i % 2 else math.sqrt(0.5 * (1 - rng.uniform(-1, 1)))
        lam = rng.uniform(0.2, 5.0) if i % 3 else 12398.419843 / rng.uniform(4000, 15000)
        inv = 1.0 / lam
        q0 = x * inv
        r = float(Fraction(x) - Fraction(q0) * Fraction(lam))
        q = float(Fraction(r) * Fraction(inv) + Fraction(q0))
        assert q == x / lam, (x, lam)


def test_write_image_bytes_equal_reference(tmp_path):
    """write_image (io.py:403-434): the .bin payload and the .json sidecar text equal, byte for
    byte, what the reference's write_image wrote for the same accumulator and metadata
    (tests/golden/image_io.npz)."""
    from paper_2205_07976_b200 import BeamSpectrum, DetectorPanel, PixelBuffer
    from paper_2205_07976_b200.io import read_image, write_image

    case = np.load(parity.GOLDEN / "image_io.npz")
    panel = DetectorPanel(24, 40, 88.6e-6, 0.1417, (11.5, 19.5))
    spectrum = BeamSpectrum(samples=((1.7, 0.5), (1.71, 0.25), (1.72, 0.25)), fluence=1e24)
    path = write_image(PixelBuffer((24, 40), "f64", case["data"]), tmp_path / "img_000007", panel=panel,
                       spectrum=spectrum, seed=220507983, image_index=7)
    assert path.read_bytes() == case["bin"].tobytes()
    assert path.with_suffix(".json").read_text() == str(case["json"])
    data, side = read_image(path)
    assert data.shape == (24, 40) and side["image_index"] == 7


def test_ls49_edge_bright_pixels_are_conditioned_at_1e8():
    """the FP64 path's largest per-pixel difference from the reference (ls49_edge, ~6e-9 on
    pixels >= 1e-3 max; total and spots ~1e-12) is within the problem's FP64 conditioning.  The
    REFERENCE itself, with every fractional Miller index moved by one ulp inside its grating function
    (kernels.py:134-142), moves those pixels by ~1e-8 (|h| ~ 35, N = 30: N pi h ~ 3300 rad), while its
    total and spots move by ~1e-12 (tools/conditioning.py).  Needs the reference (this container)."""
    import sys
    from pathlib import Path

    if not Path("/root/reference/pkg/src").exists():
        pytest.skip("reference package not present (it never is on the GPU box)")
    sys.path.insert(0, str(Path(__file__).resolve().parents[1] / "tools"))
    import conditioning

    case = parity.load("ls49_edge")
    img = conditioning.run(case, 1)
    m = parity.metrics(img, case["ref_f64"], (int(case["panel"][0]), int(case["panel"][1])))
    assert m["pix_rel_bright"] > 6e-9, m   # the reference against itself, one ulp of h apart
    assert m["total"] < 1e-11 and m["spot"] < 1e-11, m
