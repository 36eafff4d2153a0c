"""Seeded random configurations through the drop-in API vs the CPU oracle (both paths).

Each case draws a triclinic cell and orientation, a tilted / off-axis panel (sometimes a
two-panel detector with thickness layers), a spectrum that is uniform in 1/lambda or random,
mosaic domains, oversampling, crystal size, Fhkl table, shape transform and phi scan, so the
plan's choices -- FP32
MUFU vs polynomial numerator, FP32 chunking, FP64 recurrence runs vs direct kernel, dense
vs sparse Fhkl, row-banded host download -- are all exercised against the same independent
checker.  Tolerances: FP64 1e-9, FP32 1e-4 on total and every spot.
"""
import dataclasses
import math

import numpy as np
import pytest

import parity
from oracle import oracle
from paper_2205_07976_b200 import (BeamSpectrum, CrystalModel, Detector, DetectorPanel, Orientation, PhiScan, PixelBuffer,
                                   SpotsContext, SpotsPlan, StructureFactorTable, UnitCell, describe,
                                   generate_mosaic_rotations, nanobragg_spots, synthetic)

pytestmark = pytest.mark.gpu

HC = 12398.419843


def random_case(seed: int) -> SpotsContext:
    rng = np.random.default_rng(1000 + seed)
    while True:
        try:
            cell = UnitCell(*rng.uniform(20, 90, 3), *rng.uniform(70, 115, 3))
            break
        except Exception:
            continue
    u = synthetic.random_rotation(rng)
    n_cells = tuple(int(x) for x in rng.integers(3, 25, 3))
    n_dom = int(rng.integers(1, 9))
    mosaic = generate_mosaic_rotations(seed, float(rng.uniform(0.0, 0.3)), n_dom)
    dmin = 2.5
    table = synthetic.wilson_table(cell, dmin, seed, f000=float(rng.uniform(0, 500)))
    if rng.random() < 0.3:  # a sparse table with a non-zero default amplitude
        table = StructureFactorTable(dict(list(table.entries.items())[::7]), float(rng.uniform(0, 50)))
    crystal = CrystalModel(cell, Orientation(u), n_cells, mosaic, table)
    n_src = int(rng.integers(1, 40))
    if rng.random() < 0.6:  # uniform in energy (1/lambda): the FP64 recurrence runs
        e = float(rng.uniform(6000, 9000)) + float(rng.uniform(0.1, 3.0)) * np.arange(n_src)
    else:
        e = rng.uniform(6000, 9000, n_src)
    spec = BeamSpectrum(samples=tuple(zip((HC / e).tolist(), rng.uniform(0.1, 1.0, n_src).tolist())),
                        fluence=1e24, polarization_on=bool(rng.random() < 0.7))
    ang = float(rng.uniform(-0.4, 0.4))
    fast = (math.cos(ang), math.sin(ang), 0.0)
    slow = (-math.sin(ang), math.cos(ang), 0.0)
    rows, cols = int(rng.integers(8, 40)), int(rng.integers(8, 40))
    px = float(rng.uniform(70e-6, 180e-6))
    bc = (float(rng.uniform(-600, 600)), float(rng.uniform(-600, 600)))
    dist = float(rng.uniform(0.08, 0.25))
    if rng.random() < 0.3:
        thick = float(rng.uniform(100e-6, 450e-6))
        panels = tuple(DetectorPanel(rows, cols, px, dist, (bc[0] - k * (rows + 3), bc[1]), fast_axis=fast,
                                     slow_axis=slow, thickness=thick, thick_steps=int(rng.integers(1, 4)),
                                     attenuation_length=60e-6) for k in range(2))
        panel = Detector(panels)
    else:
        panel = DetectorPanel(rows, cols, px, dist, bc, fast_axis=fast, slow_axis=slow)
    shape = "sincg" if rng.random() < 0.75 else str(rng.choice(["gauss", "round", "tophat"]))
    phi = PhiScan(float(rng.uniform(-5, 5)), float(rng.uniform(0, 0.5)), int(rng.integers(1, 4)),
                  tuple(synthetic.random_rotation(rng)[0])) if rng.random() < 0.25 else None
    return SpotsContext(crystal, panel, spec, oversample=int(rng.integers(1, 4)), shape=shape, phi=phi)


@pytest.mark.parametrize("seed", range(int(__import__("os").environ.get("NBX_FUZZ_CASES", "32"))))
def test_random_configuration_vs_oracle(gpu, seed):
    ctx = random_case(seed)
    want, _ = oracle.spots(describe(ctx), "f64")
    for compute, tol in (("fp64", 1e-9), ("fp32", 1e-4)):
        c = dataclasses.replace(ctx, compute=compute)
        out = PixelBuffer.zeros(c.panel.dims, "f64")
        nanobragg_spots(c, out)
        info = SpotsPlan(c).info
        if compute == "fp32" and want.sum() < 1e-30:
            # physically empty image (e.g. a Gaussian transform far from every lattice point:
            # ~1e-96 photons): below FP32's range relative to the sigma-scaled peak the FP32
            # path returns ~0; only the absolute agreement is meaningful there
            assert np.abs(out.data - want).max() < 1e-30, (seed, info.kernel_variant)
            continue
        m = parity.metrics(out.data, want, c.panel.dims)
        assert m["total"] < tol and m["spot"] < tol, (compute, seed, info.kernel_variant, info.table_kind, m)


@pytest.mark.parametrize("seed", range(12))
def test_random_channel_shards_sum_to_whole(gpu, seed):
    """The channel-sharded decomposition (C5) on random configurations: FP64 partials of random
    source shards, summed and scaled once, equal the whole image (both paths)."""
    from paper_2205_07976_b200 import _native as N

    ctx = random_case(100 + seed)
    n_src = len(ctx.spectrum.samples)
    if n_src < 2:
        pytest.skip("one source")
    cut = int(np.random.default_rng(seed).integers(1, n_src))
    for compute, rtol in (("fp64", 1e-11), ("fp32", 1e-4)):
        c = dataclasses.replace(ctx, compute=compute)
        whole = PixelBuffer.zeros(c.panel.dims, "f64")
        nanobragg_spots(c, whole)
        if compute == "fp32" and whole.data.sum() < 1e-30:
            continue  # physically empty image (see test_random_configuration_vs_oracle)
        plan = SpotsPlan(c)
        raw = np.zeros(plan.n_pixels)
        for lo, hi in ((0, cut), (cut, n_src)):
            SpotsPlan(c, src_begin=lo, src_end=hi, norm=0.0).run(raw, mode=N.OUT_RAW_F64)
        got = raw * plan.scale
        m = parity.metrics(got, whole.data, c.panel.dims)
        assert m["total"] < rtol and m["spot"] < rtol, (compute, seed, cut, m)
