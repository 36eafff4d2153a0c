"""Host-side setup types (model.py) against the reference's semantics (CPU only).

Two layers:
  * known answers that hold for any faithful implementation (the reference's own
    test_model.py cases, restated): cell validation and volume, basis conventions and
    duality, proper rotations, mosaic generator determinism, half-away rounding and the
    default amplitude, panel/spectrum/profile validation, solid angle and polarization;
  * a differential check against the reference package itself, when it is importable in
    this container (/root/reference/pkg/src; skipped elsewhere): the same inputs give
    bit-identical bases, mosaic rotations, lab positions, solid angles, Miller indices,
    Fhkl lookups and background interpolation, and the same invalid inputs raise errors of
    the same class names.
"""
import math
import sys
from pathlib import Path

import numpy as np
import pytest

from paper_2205_07976_b200 import (BackgroundProfile, BeamSpectrum, CrystalModel, DetectorPanel, MosaicDomainSet,
                                   Orientation, StructureFactorTable, UnitCell, generate_mosaic_rotations)
from paper_2205_07976_b200 import model as mm

REF_SRC = Path("/root/reference/pkg/src")


def ref():
    if not REF_SRC.exists():
        pytest.skip("reference package not present (it never is on the GPU box)")
    if str(REF_SRC) not in sys.path:
        sys.path.insert(0, str(REF_SRC))
    import xtrace.model as xm

    return xm


# --------------------------------------------------------------------------- known answers

@pytest.mark.parametrize("args", [(0, 1, 1, 90, 90, 90), (1, -2, 1, 90, 90, 90), (1, 1, 1, 0, 90, 90),
                                  (1, 1, 1, 90, 180, 90), (1, 1, 1, 10, 10, 170)])
def test_cell_validation(args):
    with pytest.raises(mm.InvalidCellError):
        UnitCell(*args)


def test_cell_volume_and_basis_conventions():
    assert UnitCell(2, 3, 4, 90, 90, 90).volume() == pytest.approx(24.0, rel=1e-15)
    b = mm.real_basis(UnitCell(10, 20, 30, 80, 95, 105))
    assert b[0, 1] == b[0, 2] == b[1, 2] == 0.0  # a along x, b in the x-y plane
    rng = np.random.default_rng(3)
    for _ in range(20):
        cell = UnitCell(*rng.uniform(5, 80, 3), *rng.uniform(70, 110, 3))
        a, r = mm.real_basis(cell), mm.reciprocal_basis(cell)
        np.testing.assert_allclose(a @ r.T, np.eye(3), atol=1e-13)


def test_orientation_must_be_proper_rotation():
    with pytest.raises(mm.GeometryError):
        Orientation(np.diag([1.0, 1.0, 1.1]))
    with pytest.raises(mm.GeometryError):
        Orientation(np.diag([1.0, 1.0, -1.0]))
    np.testing.assert_array_equal(Orientation().u, np.eye(3))


def test_mosaic_generator():
    z = generate_mosaic_rotations(7, 0.0, 5)
    np.testing.assert_array_equal(z.rotations, np.broadcast_to(np.eye(3), (5, 3, 3)))
    a, b = generate_mosaic_rotations(11, 0.5, 20), generate_mosaic_rotations(11, 0.5, 20)
    np.testing.assert_array_equal(a.rotations, b.rotations)
    assert not np.array_equal(a.rotations, generate_mosaic_rotations(12, 0.5, 20).rotations)
    for r in a.rotations:
        np.testing.assert_allclose(r @ r.T, np.eye(3), atol=1e-14)
        assert np.linalg.det(r) == pytest.approx(1.0, abs=1e-14)
    with pytest.raises(ValueError):
        generate_mosaic_rotations(1, 0.1, 0)


def test_fhkl_half_away_rounding_and_default():
    t = StructureFactorTable({(1, 0, 0): 10.0, (-1, 0, 0): 20.0, (2, 0, 0): 30.0, (-3, 0, 0): 40.0}, default_f=5.0)
    assert [mm.round_half_away(x) for x in (0.5, -0.5, 1.5, -2.5, 0.49999999)] == [1, -1, 2, -3, 0]
    assert mm.lookup_f(t, 0.5, 0.2, -0.4) == 10.0
    assert mm.lookup_f(t, -0.5, 0.0, 0.0) == 20.0
    assert mm.lookup_f(t, 1.5, 0.0, 0.0) == 30.0
    assert mm.lookup_f(t, -2.5, 0.0, 0.0) == 40.0
    assert mm.lookup_f(t, 7.2, 1.0, 1.0) == 5.0
    with pytest.raises(ValueError):
        StructureFactorTable({(0, 0, 0): -1.0})


def test_panel_spectrum_profile_validation():
    with pytest.raises(mm.GeometryError):
        DetectorPanel(4, 4, 1e-4, 0.1, (1.5, 1.5), fast_axis=(1.0, 0.0, 0.0), slow_axis=(1.0, 0.0, 0.0))
    with pytest.raises(mm.GeometryError):
        DetectorPanel(4, 4, 1e-4, 0.1, (1.5, 1.5), fast_axis=(2.0, 0.0, 0.0))
    with pytest.raises((mm.GeometryError, ValueError)):
        DetectorPanel(0, 4, 1e-4, 0.1, (1.5, 1.5))
    with pytest.raises(ValueError):
        BeamSpectrum(samples=((1.0, 0.0),), fluence=1e24)
    with pytest.raises(ValueError):
        BeamSpectrum(samples=((-1.0, 1.0),), fluence=1e24)
    with pytest.raises(ValueError):
        BackgroundProfile(points=((0.2, 1.0), (0.1, 2.0)))
    prof = BackgroundProfile(points=((0.0, 1.0), (0.2, 3.0), (0.4, 2.0)))
    assert mm.interp_background_f(prof, 0.1) == 2.0
    assert mm.interp_background_f(prof, 0.0) == 1.0 and mm.interp_background_f(prof, 9.0) == 2.0


def test_solid_angle_and_polarization():
    panel = DetectorPanel(4, 4, 100e-6, 0.1, (1.5, 1.5))
    on_axis = mm.solid_angle(panel, (0.0, 0.0, 0.1))
    assert on_axis == pytest.approx((100e-6) ** 2 / 0.01, rel=1e-15)
    assert mm.solid_angle(panel, (0.0, 0.0, 0.2)) * 4 == pytest.approx(on_axis, rel=1e-15)  # inverse square
    spec = BeamSpectrum(samples=((1.0, 1.0),), fluence=1e24, polarization_on=True)
    assert mm.polarization_factor(spec, 0.0) == 1.0
    assert mm.polarization_factor(spec, math.pi / 2) == pytest.approx(0.5, abs=1e-16)
    assert mm.polarization_factor(BeamSpectrum(samples=((1.0, 1.0),), fluence=1e24, polarization_on=False), 1.0) == 1.0


# --------------------------------------------------------------------------- differential vs the reference

def test_bases_and_mosaic_bitwise_equal_reference():
    xm = ref()
    rng = np.random.default_rng(5)
    for _ in range(30):
        p = (*rng.uniform(5, 90, 3), *rng.uniform(60, 120, 3))
        try:
            rc = xm.UnitCell(*p)
        except Exception as e:  # same invalid inputs must fail here too
            with pytest.raises(Exception) as ours:
                UnitCell(*p)
            assert type(ours.value).__name__ == type(e).__name__
            continue
        c = UnitCell(*p)
        np.testing.assert_array_equal(mm.real_basis(c), xm.real_basis(rc))
        np.testing.assert_array_equal(mm.reciprocal_basis(c), xm.reciprocal_basis(rc))
        assert c.volume() == rc.volume()
    for seed, spread, n in ((1, 0.05, 50), (220507976, 0.2, 7), (3, 1.0, 3)):
        np.testing.assert_array_equal(generate_mosaic_rotations(seed, spread, n).rotations,
                                      xm.generate_mosaic_rotations(seed, spread, n).rotations)


def test_geometry_and_lookup_bitwise_equal_reference():
    xm = ref()
    rng = np.random.default_rng(9)
    ang = math.radians(20.0)
    fast = (math.cos(ang), math.sin(ang), 0.0)
    slow = (-math.sin(ang), math.cos(ang), 0.0)
    ours = DetectorPanel(64, 48, 88.6e-6, 0.1417, (31.5, 20.25), fast_axis=fast, slow_axis=slow)
    theirs = xm.DetectorPanel(64, 48, 88.6e-6, 0.1417, (31.5, 20.25), fast_axis=fast, slow_axis=slow)
    beam = (0.0, 0.0, 1.0)
    for _ in range(40):
        s, f = int(rng.integers(0, 64)), int(rng.integers(0, 48))
        ss, sf = float(rng.random()), float(rng.random())
        p = mm.pixel_lab_position(ours, s, f, ss, sf, beam)
        np.testing.assert_array_equal(p, xm.pixel_lab_position(theirs, s, f, ss, sf, beam))
        assert mm.solid_angle(ours, p) == xm.solid_angle(theirs, p)
    entries = {tuple(int(v) for v in rng.integers(-6, 7, 3)): float(rng.uniform(0, 100)) for _ in range(80)}
    t, rt = StructureFactorTable(entries, 3.5), xm.StructureFactorTable(entries, 3.5)
    h, k, l = (rng.uniform(-7, 7, 500) for _ in range(3))
    h[:5] = [0.5, -0.5, 2.5, -3.5, 1e7]  # ties and an out-of-range index
    np.testing.assert_array_equal(t.lookup_rounded(h, k, l), rt.lookup_rounded(h, k, l))
    cell = UnitCell(67.2, 59.8, 47.2, 90, 113.2, 90)
    mos = generate_mosaic_rotations(4, 0.1, 3)
    u = np.linalg.qr(rng.normal(size=(3, 3)))[0]
    u *= np.sign(np.linalg.det(u))
    cm = CrystalModel(cell, Orientation(u), (10, 10, 10), MosaicDomainSet(mos.rotations), t)
    rcm = xm.CrystalModel(xm.UnitCell(67.2, 59.8, 47.2, 90, 113.2, 90), xm.Orientation(u), (10, 10, 10),
                          xm.MosaicDomainSet(mos.rotations), rt)
    np.testing.assert_array_equal(cm.rotated_real_bases(), rcm.rotated_real_bases())
    for m in range(3):
        q = rng.normal(size=3)
        assert mm.fractional_miller(cm, m, q) == xm.fractional_miller(rcm, m, q)


def test_background_interp_and_validation_equal_reference():
    xm = ref()
    pts = ((0.0, 2.57), (0.0365, 2.58), (0.07, 2.8), (0.12, 5.0), (0.162, 8.0), (0.3, 6.5))
    ours, theirs = BackgroundProfile(points=pts), xm.BackgroundProfile(points=pts)
    for x in np.linspace(0.0, 0.5, 101):
        assert mm.interp_background_f(ours, float(x)) == xm.interp_background_f(theirs, float(x))
    for bad in (((0.1, 1.0), (0.1, 2.0)), ((0.0, -1.0), (0.1, 1.0))):
        with pytest.raises(Exception) as e_ref:
            xm.BackgroundProfile(points=bad)
        with pytest.raises(Exception) as e_ours:
            BackgroundProfile(points=bad)
        assert type(e_ours.value).__name__ == type(e_ref.value).__name__


def test_public_names_cover_the_reference_spot_api():
    """Every public name of xtrace.model / xtrace.kernels exists here (DESIGN.md §9 lists the
    out-of-scope top-level names, which are the only ones allowed to be missing)."""
    ref()
    import xtrace
    import xtrace.kernels as xk
    import xtrace.model as xm

    import paper_2205_07976_b200 as ours
    import paper_2205_07976_b200.kernels as ok

    assert not set(xm.__all__) - set(dir(mm))
    assert not {n for n in xk.__all__ if not hasattr(ok, n)}
    out_of_scope = {"CampaignIOError", "CampaignPlan", "CampaignReport", "ConfigError", "ParseError", "RangePolicy",
                    "ScalingRow", "SimulationConfig", "default_worker_count", "kernel_time_table", "load_background",
                    "load_config", "load_hkl", "parallel_for", "parallel_reduce", "parallel_scan", "scheduler",
                    "strong_scaling", "write_preview", "write_scaling_csv"}
    public = {n for n in dir(xtrace) if not n.startswith("_")}
    assert public - set(dir(ours)) <= out_of_scope, sorted(public - set(dir(ours)) - out_of_scope)
