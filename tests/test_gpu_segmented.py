"""The segmented FP64 channel recurrence (kernel variant 6, nbx_kernels.cu:domain_sum_f64_cap).

Per run the kernel predicts, in FP32, the channel at which each axis's Fhkl index changes and
the channels that sit within the margins of a half-integer (index not provable) or within
|sin(pi h)| < ~1e-4 of a Bragg position (evaluated exactly); everything else runs the bare
recurrence.  These tests aim at the prediction's corners -- index changes in the first and
last channels, two axes changing together, steps far below the margins (the direct beam),
spans that force several runs -- and compare the image with the direct per-channel FP64
kernel (variant 0, no prediction at all) and with the CPU oracle.
"""
import dataclasses

import numpy as np
import pytest

import parity
from oracle import oracle
from paper_2205_07976_b200 import (BeamSpectrum, CrystalModel, DetectorPanel, MosaicDomainSet, Orientation,
                                   PixelBuffer, SpotsContext, SpotsPlan, StructureFactorTable, UnitCell, describe,
                                   nanobragg_spots, synthetic)
from paper_2205_07976_b200 import _native as N

pytestmark = pytest.mark.gpu
HC = 12398.419843


def image(ctx, monkeypatch, rec=None):
    if rec is None:
        monkeypatch.delenv("NBX_FP64_REC", raising=False)
    else:
        monkeypatch.setenv("NBX_FP64_REC", rec)
    plan = SpotsPlan(ctx)
    out = np.zeros(plan.n_pixels)
    plan.run(out, mode=N.OUT_F64)
    info = plan.info
    plan.close()
    monkeypatch.delenv("NBX_FP64_REC", raising=False)
    return out, info


def uniform_spectrum(e0, de, n, seed=3):
    e = e0 + de * np.arange(n)
    w = np.random.default_rng(seed).uniform(0.2, 1.0, n)
    return BeamSpectrum(samples=tuple(zip((HC / e).tolist(), w.tolist())), fluence=1e24, polarization_on=True)


def check_against_direct(ctx, monkeypatch, tol=1e-11):
    seg, info = image(ctx, monkeypatch)
    assert info.kernel_variant == 6 and info.channel_runs >= 1, (info.kernel_variant, info.channel_runs)
    direct, dinfo = image(ctx, monkeypatch, "0")
    assert dinfo.kernel_variant == 0
    m = parity.metrics(seg, direct, ctx.panel.dims)
    assert m["total"] < tol and m["spot"] < tol and m["pix_abs_over_max"] < 10 * tol, m
    return seg, info


@pytest.mark.parametrize("seed", range(8))
def test_segmented_vs_direct_random_wide_band(gpu, monkeypatch, seed):
    """Random triclinic crystals, high resolution (|h| up to ~45) and wide uniform bands
    (several index changes per axis per run -> the host's 0.9 phase-span rule cuts runs)."""
    rng = np.random.default_rng(50 + seed)
    cell = UnitCell(*rng.uniform(35, 80, 3), *rng.uniform(80, 110, 3))  # uniform-run check: |S| dev <= 1e-14
    table = synthetic.wilson_table(cell, 1.8, seed, f000=300.0)
    crystal = CrystalModel(cell, Orientation(synthetic.random_rotation(rng)),
                           tuple(int(x) for x in rng.integers(5, 40, 3)),
                           synthetic.generate_mosaic_rotations(seed, 0.2, 3), table)
    n = int(rng.integers(20, 160))
    # widest step that keeps the mean run >= 8 channels under the span rule (|S| <= 2 max edge)
    de_max = 0.9 * HC / (8 * 2 * max(cell.a, cell.b, cell.c))
    spec = uniform_spectrum(float(rng.uniform(6500, 9000)), float(rng.uniform(0.3, 1.0)) * de_max, n, seed)
    r0, c0 = int(rng.integers(0, 3800)), int(rng.integers(0, 3800))
    panel = synthetic.roi(synthetic.rayonix_panel(), r0, c0, 24, 40)
    ctx = SpotsContext(crystal, panel, spec, oversample=int(rng.integers(1, 3)), compute="fp64")
    _, info = check_against_direct(ctx, monkeypatch)
    want, _ = oracle.spots(describe(ctx), "f64")
    got = PixelBuffer.zeros(panel.dims, "f64")
    nanobragg_spots(ctx, got)
    m = parity.metrics(got.data, want, panel.dims)
    assert m["total"] < 1e-9 and m["spot"] < 1e-9, m


def test_span_rule_cuts_runs(gpu, monkeypatch):
    """A 200 eV band over 100 channels (2 eV steps): |Delta| * 99 > 0.9 at the edge of the detector, so the
    100 channels are split into several runs, each with at most one index change per axis."""
    panel = synthetic.roi(synthetic.rayonix_panel(), 0, 0, 16, 48)
    ctx = dataclasses.replace(synthetic.ls49_context(panel=panel, n_domains=2, compute="fp64"),
                              spectrum=uniform_spectrum(7000.0, 2.0, 100))
    _, info = check_against_direct(ctx, monkeypatch)
    assert info.channel_runs >= 2


def test_direct_beam_exact_bragg_and_tiny_steps(gpu, monkeypatch):
    """The pixel centred on the beam has S = 0 on every axis: h = 0 for every channel, steps
    of exactly zero, every channel slow and the reference's limit branch (F000, N^3 peak).
    Its neighbours have |Delta| ~ 5e-6 per channel, the size of the prediction margins."""
    cell = UnitCell(60.0, 60.0, 60.0, 90.0, 90.0, 90.0)
    table = StructureFactorTable({(0, 0, 0): 400.0, (1, 0, 0): 90.0}, default_f=5.0)
    crystal = CrystalModel(cell, Orientation(), (7, 9, 11), MosaicDomainSet(np.eye(3)[None]), table)
    panel = DetectorPanel(9, 9, 100e-6, 0.1, (4.5, 4.5))  # beam through the centre of pixel (4, 4)
    ctx = SpotsContext(crystal, panel, uniform_spectrum(8000.0, 1.0, 64), compute="fp64")
    seg, _ = check_against_direct(ctx, monkeypatch, tol=1e-11)
    want, _ = oracle.spots(describe(ctx), "f64")
    m = parity.metrics(seg, want, panel.dims)
    assert m["total"] < 1e-9 and m["spot"] < 1e-9, m
    assert np.argmax(seg) == 4 * 9 + 4


def test_index_changes_at_first_and_last_channel(gpu, monkeypatch):
    """Scan the band edge across a half-integer: for a row of pixels the index of one axis
    changes exactly between channels 0/1, in the middle and between the last two channels."""
    cell = UnitCell(80.0, 80.0, 80.0, 90.0, 90.0, 90.0)
    table = synthetic.wilson_table(cell, 2.0, 5, f000=100.0)
    rot = synthetic.random_rotation(np.random.default_rng(9))
    crystal = CrystalModel(cell, Orientation(rot), (20, 20, 20), MosaicDomainSet(np.eye(3)[None]), table)
    panel = DetectorPanel(4, 512, 100e-6, 0.08, (-300.0, -200.0))
    for de in (0.5, 3.0, 12.0):
        ctx = SpotsContext(crystal, panel, uniform_spectrum(7500.0, de, 41), compute="fp64")
        check_against_direct(ctx, monkeypatch)


def test_two_axes_change_together(gpu, monkeypatch):
    """A cubic cell along the diagonal: h and k are equal for every pixel of the diagonal, so
    their indices change at the same channel (the event loop handles both at once)."""
    cell = UnitCell(50.0, 50.0, 50.0, 90.0, 90.0, 90.0)
    table = synthetic.wilson_table(cell, 2.0, 8, f000=50.0)
    crystal = CrystalModel(cell, Orientation(), (15, 15, 15), MosaicDomainSet(np.eye(3)[None]), table)
    panel = DetectorPanel(64, 64, 150e-6, 0.07, (-100.0, -100.0),
                          fast_axis=(1.0, 0.0, 0.0), slow_axis=(0.0, 1.0, 0.0))
    ctx = SpotsContext(crystal, panel, uniform_spectrum(8000.0, 6.0, 60), compute="fp64")
    check_against_direct(ctx, monkeypatch)


def test_c2_takes_the_segmented_kernel(gpu):
    info = SpotsPlan(synthetic.ls49_context(compute="fp64")).info
    assert info.kernel_variant == 6 and info.channel_runs == 1


@pytest.mark.parametrize("seed", [0, 1])
def test_fp32_segmented_indices_opt_in(gpu, monkeypatch, seed):
    """The opt-in FP32 loop with segmented indices (variant 7, NBX_FP32_SEG=1) gives the
    per-channel loop's indices and reduced phases exactly -- only where F^2 multiplies differs
    (1e-6) -- and matches the oracle at the FP32 tolerance, on LS49 ROIs and a wide band."""
    from paper_2205_07976_b200 import _native as N

    for r0, c0, de in ((1888, 1888, 1.0), (40, 3700, 1.0), (600, 900, 3.0)):
        panel = synthetic.roi(synthetic.rayonix_panel(), r0, c0, 32, 48)
        ctx = synthetic.ls49_context(synthetic.SEED + seed, panel=panel, de=de, compute="fp32")
        imgs = {}
        for env in ("1", "0"):
            monkeypatch.setenv("NBX_FP32_SEG", env)
            plan = SpotsPlan(ctx)
            assert plan.info.kernel_variant == (7 if env == "1" else 1)
            out = np.zeros(plan.n_pixels)
            plan.run(out, mode=N.OUT_F64)
            plan.close()
            imgs[env] = out
        monkeypatch.delenv("NBX_FP32_SEG")
        m = parity.metrics(imgs["1"], imgs["0"], panel.dims)
        assert m["total"] < 1e-6 and m["spot"] < 1e-6, m
        want, _ = oracle.spots(describe(ctx), "f64")
        m = parity.metrics(imgs["1"], want, panel.dims)
        assert m["total"] < 1e-4 and m["spot"] < 1e-4, m


def test_full_shard_of_short_runs(gpu, monkeypatch):
    """8192 sources (one launch's maximum) in uniform runs of 16 channels separated by gaps -- near
    the largest shared-memory footprint of the segmented kernel (channels, >= 512 runs, event
    records; the plan needs a mean run of >= 8) -- and in runs of 128: the plan keeps variant 6 and
    the image equals the direct kernel's."""
    rng = np.random.default_rng(8192)
    cell = UnitCell(28.0, 31.0, 35.0, 90.0, 97.0, 90.0)  # small cell: the uniform-run check holds at rounding
    crystal = CrystalModel(cell, Orientation(synthetic.random_rotation(rng)), (12, 14, 10),
                           synthetic.generate_mosaic_rotations(5, 0.1, 1), synthetic.wilson_table(cell, 2.0, 5))
    panel = synthetic.roi(synthetic.rayonix_panel(), 900, 1100, 8, 32)
    for run_len in (16, 128):
        n_runs = 8192 // run_len
        e = (7000.0 + 0.01 * np.arange(run_len))[None, :] + 3.0 * np.arange(n_runs)[:, None]
        w = rng.uniform(0.2, 1.0, e.size)
        spec = BeamSpectrum(samples=tuple(zip((HC / e.ravel()).tolist(), w.tolist())), fluence=1e24,
                            polarization_on=True)
        ctx = SpotsContext(crystal, panel, spec, compute="fp64")
        got, info = image(ctx, monkeypatch)
        assert info.kernel_variant == 6 and info.channel_runs >= n_runs, (run_len, info.kernel_variant,
                                                                          info.channel_runs)
        direct, _ = image(ctx, monkeypatch, "0")
        m = parity.metrics(got, direct, panel.dims)
        assert m["total"] < 1e-11 and m["spot"] < 1e-11, (run_len, m)
