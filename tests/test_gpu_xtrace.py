"""The drop-in inside the reference's OWN pipeline.

Imports the unmodified reference package (baseline/_ref/xtrace, installed by
`pip install --target baseline/_ref`; it travels to the GPU box with the repo),
replaces its spot and background kernels with this package's drop-ins exactly as the
INTEGRATION.md shim does (the reference scheduler binds the names at import, so the
scheduler module's references are the ones that matter, scheduler.py:25), and runs:

  * xtrace.scheduler.simulate_image (scheduler.py:156-183) on the reference's small
    scheduler config: accumulators equal the reference-run fixture (sim_config.npz), and
    the executor's log holds the reference's own records -- ONE nanobragg_spots per image
    (kernel_timer, execution.py:350-356; the drop-in logs nothing itself);
  * xtrace.scheduler._rank_task (scheduler.py:190-247) on an image set that overflows
    float32: every image is FLAGGED with the reference's lowest bad pixel (the drop-in
    raises xtrace.errors.PatternFault / NumericalFault, which _rank_task catches at
    :212), the rank reports no error, and the flagged list equals the unpatched
    reference's own;
  * the error classes on bad dims: xtrace.errors.ShapeMismatchError.
"""
from __future__ import annotations

import contextlib
import sys
import threading
from pathlib import Path

import numpy as np
import pytest

import parity

REF = Path(__file__).resolve().parents[1] / "baseline" / "_ref"
pytestmark = [pytest.mark.gpu,
              pytest.mark.skipif(not (REF / "xtrace" / "kernels.py").exists(),
                                 reason="reference install baseline/_ref absent (DESIGN.md §10)")]


@pytest.fixture(scope="module")
def xtrace():
    if str(REF) not in sys.path:
        sys.path.insert(0, str(REF))
    import xtrace  # noqa: F401
    import xtrace.errors
    import xtrace.execution
    import xtrace.io
    import xtrace.kernels
    import xtrace.model
    import xtrace.scheduler

    return sys.modules["xtrace"]


@pytest.fixture
def patched(xtrace, monkeypatch, gpu):
    """The INTEGRATION.md shim: xtrace's spot and background kernels -> the B200 drop-ins."""
    import paper_2205_07976_b200 as nbx

    for mod in (xtrace.kernels, xtrace.scheduler):
        monkeypatch.setattr(mod, "nanobragg_spots", nbx.nanobragg_spots)
        monkeypatch.setattr(mod, "add_background", nbx.add_background)
    return xtrace


def small_config(xtrace, fluence=1e24, default_f=100.0):
    xm, xio = xtrace.model, xtrace.io
    # test_scheduler.py:30-45 of the reference (the config of tests/golden/sim_config.npz)
    return xio.SimulationConfig(
        cell=xm.UnitCell(100.0, 100.0, 100.0, 90.0, 90.0, 90.0), n_cells=(5, 5, 5),
        panel=xm.DetectorPanel(48, 48, 100e-6, 0.1, (23.5, 23.5)),
        spectrum=xm.BeamSpectrum(samples=((1.0, 1.0),), fluence=fluence),
        sf_table=xm.StructureFactorTable({}, default_f=default_f),
        background=xm.BackgroundProfile(points=((0.0, 2.57), (0.07, 2.8), (0.3, 6.5))),
        mosaic_domains=2, mosaic_spread_deg=0.05, oversample=1, seed=0)


def test_reference_simulate_image_through_drop_in(patched):
    xs = patched.scheduler
    case = np.load(parity.GOLDEN / "sim_config.npz")
    config = small_config(patched)
    ex = patched.execution.Executor.serial()
    for seed, want in zip(case["seeds"], case["ref_images"]):
        got = xs.simulate_image(config, int(seed), ex)
        assert type(got).__module__ == "xtrace.kernels" and got.precision == "f64"
        # f64(f32(spots)) + f64(f32(background)): each staged term within one f32 ulp
        np.testing.assert_allclose(got.data, want, rtol=2.0 ** -22, atol=0)
    labels = [r.label for r in ex.timing_log]
    n = len(case["seeds"])
    assert labels.count("nanobragg_spots") == n, labels
    assert labels.count("add_background") == n, labels
    assert labels == ["nanobragg_spots", "add_array", "add_background", "add_array"] * n


def _rank(xtrace, config, n):
    xs = xtrace.scheduler
    plan = xs.CampaignPlan(n_images=n, seed=0)
    return xs._rank_task(0, (0, n), config, plan, None, True, "serial", 1, contextlib.nullcontext(),
                         threading.Event())


def test_rank_task_flags_overflow_images_like_the_reference(xtrace, monkeypatch, gpu):
    """A float32-overflowing image is flagged (index, lowest bad pixel), not a rank error."""
    import paper_2205_07976_b200 as nbx

    config = small_config(xtrace, fluence=1e24, default_f=1e23)  # some pixels overflow f32 (first: 99)
    want = _rank(xtrace, config, 2)  # the unpatched reference (NumPy) on the same images
    assert want["error"] is None and len(want["flagged"]) == 2, want["flagged"]
    for mod in (xtrace.kernels, xtrace.scheduler):
        monkeypatch.setattr(mod, "nanobragg_spots", nbx.nanobragg_spots)
        monkeypatch.setattr(mod, "add_background", nbx.add_background)
    got = _rank(xtrace, config, 2)
    assert got["error"] is None, got["error"]
    assert got["flagged"] == want["flagged"]
    assert not got["images"]  # flagged images are skipped, as in the reference
    # a healthy config through the same rank loop: nothing flagged, one spot record per image
    ok = _rank(xtrace, small_config(xtrace), 3)
    assert ok["error"] is None and ok["flagged"] == [] and sorted(ok["images"]) == [0, 1, 2]
    assert [r.label for r in ok["timing"]].count("nanobragg_spots") == 3


def test_reference_error_classes(xtrace, gpu):
    """xtrace objects in -> xtrace.errors classes out, with the reference's lowest bad pixel."""
    import paper_2205_07976_b200 as nbx
    from paper_2205_07976_b200 import errors as ours

    xk, xe = xtrace.kernels, xtrace.errors
    config = small_config(xtrace, default_f=6e22)
    ctx = xk.SpotsContext(config.crystal_for_seed(3), config.panel, config.spectrum, 1)
    with pytest.raises(xe.PatternFault) as ref:  # the unpatched reference body (kernels.py:211-216)
        xk.nanobragg_spots(ctx, xk.PixelBuffer.zeros(config.panel.dims, "f32"))
    with pytest.raises(xe.ShapeMismatchError):
        nbx.nanobragg_spots(ctx, xk.PixelBuffer.zeros((47, 48), "f32"))
    out = xk.PixelBuffer.zeros(config.panel.dims, "f32")
    with pytest.raises(xe.PatternFault) as got:
        nbx.nanobragg_spots(ctx, out)
    assert isinstance(got.value.cause, xe.NumericalFault)
    assert got.value.label == ref.value.label == "nanobragg_spots"
    assert got.value.index == ref.value.index and got.value.cause.pixel == ref.value.cause.pixel
    assert ours.hierarchy_for(ctx, out) is xe
    assert ours.hierarchy_for(object()) is ours
