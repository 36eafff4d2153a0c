"""GPU: add_background (the paper's second kernel) and the fused simulate_image accumulator."""
import numpy as np
import pytest

import parity
from oracle import oracle
from paper_2205_07976_b200 import (
    BackgroundProfile,
    PatternFault,
    PixelBuffer,
    add_array,
    add_background,
    describe,
    nanobragg_spots,
    simulate_image,
    synthetic,
)
from paper_2205_07976_b200.kernels import _bg_descriptor

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("name", ["bg_flat", "bg_scalar", "bg_water_80"])
def test_background_matches_reference(gpu, name):
    case = parity.load(name)
    prof, panel, beam, tf = parity.bg_inputs(case)
    out = PixelBuffer.zeros(panel.dims, "f64")
    add_background(prof, panel, beam, tf, out)
    np.testing.assert_allclose(out.data, case["ref_bg_f64"], rtol=1e-12, atol=0)
    out32 = PixelBuffer.zeros(panel.dims, "f32")
    add_background(prof, panel, beam, tf, out32)
    rel = np.abs(out32.data.astype(np.float64) - case["ref_bg_f32"]) / case["ref_bg_f32"]
    assert rel.max() <= 2.0 ** -23


def test_simulate_image_matches_reference_pipeline(gpu):
    """test_kernels.py:439-471 / test_acceptance.py:68-111: spots + background + add_array, 1e-6 rel per pixel."""
    case = parity.load("pipeline_full")
    prof, _, _, tf = parity.bg_inputs(case)
    img = simulate_image(parity.context(case), background=prof, thickness_factor=tf)
    rel = np.abs(img.data - case["ref_image"]) / np.abs(case["ref_image"])
    assert rel.max() < 1e-6
    # and it is exactly the staged pipeline: f64(f32 spots) + f64(f32 background)
    spots = PixelBuffer.zeros((4, 4))
    nanobragg_spots(parity.context(case), spots)
    bg = PixelBuffer.zeros((4, 4))
    add_background(prof, *parity.bg_inputs(case)[1:3], tf, bg)
    acc = PixelBuffer.zeros((4, 4), "f64")
    add_array(acc, spots)
    add_array(acc, bg)
    assert np.array_equal(img.data, acc.data)


def test_simulate_image_ls49_roi_vs_oracle(gpu):
    water = BackgroundProfile(points=((0.0, 2.57), (0.0365, 2.58), (0.07, 2.8), (0.12, 5.0), (0.162, 8.0),
                                      (0.3, 6.5)))
    panel = synthetic.roi(synthetic.rayonix_panel(), 100, 3000, 16, 64)
    for compute, tol in (("fp64", 1e-9), ("fp32", 1e-4)):
        ctx = synthetic.ls49_context(panel=panel, n_channels=12, n_domains=3, compute=compute)
        img = simulate_image(ctx, background=water, thickness_factor=0.7)
        sp, _ = oracle.spots(describe(ctx), "f64")
        bg, _ = oracle.background(_bg_descriptor(water, panel, ctx.spectrum, 0.7), "f64")
        want = sp.astype(np.float32).astype(np.float64) + bg.astype(np.float32).astype(np.float64)
        assert abs(img.data.sum() - want.sum()) / want.sum() < tol
        no_bg = simulate_image(ctx)
        assert np.allclose(no_bg.data, sp.astype(np.float32).astype(np.float64), rtol=tol)


def test_background_fault_is_labelled(gpu):
    case = parity.load("bg_scalar")
    prof, panel, beam, tf = parity.bg_inputs(case)
    with pytest.raises(PatternFault) as info:
        add_background(prof, panel, beam, 1e300, PixelBuffer.zeros(panel.dims))
    assert info.value.label == "add_background" and info.value.index == 0


@pytest.mark.parametrize("seed", range(24))
def test_background_random_profiles_vs_oracle(gpu, seed):
    """Seeded random profiles (2-40 points, some starting above or ending below the detector's
    sin(theta)/lambda range, exact hits on profile points), random spectra (unsorted, repeated
    wavelengths, zero weights) and tilted panels: the register-resident interpolation cursor
    and the 3-op division against the C restatement at 1e-12, f32 stores within 1 ulp."""
    import math

    from paper_2205_07976_b200 import BackgroundProfile, BeamSpectrum, DetectorPanel

    rng = np.random.default_rng(500 + seed)
    n_pts = int(rng.integers(2, 41))
    lo = float(rng.choice([0.0, rng.uniform(0.0, 0.3)]))
    stol = np.sort(rng.uniform(lo, lo + rng.uniform(0.05, 0.8), n_pts))
    stol = np.unique(stol)
    if stol.size < 2:
        stol = np.array([lo, lo + 0.1])
    prof = BackgroundProfile(points=tuple(zip(stol.tolist(), rng.uniform(0.0, 9.0, stol.size).tolist())))
    n_src = int(rng.integers(1, 61))
    lam = rng.uniform(0.8, 2.0, n_src)
    if n_src > 3:
        lam[1] = lam[0]  # repeated wavelength
    w = rng.uniform(0.0, 1.0, n_src)
    w[rng.random(n_src) < 0.2] = 0.0
    w[0] = max(w[0], 0.1)
    beam = BeamSpectrum(samples=tuple(zip(lam.tolist(), w.tolist())), fluence=1e24,
                        polarization_on=bool(rng.random() < 0.7))
    ang = float(rng.uniform(-0.5, 0.5))
    panel = DetectorPanel(int(rng.integers(8, 48)), int(rng.integers(8, 48)), float(rng.uniform(50e-6, 200e-6)),
                          float(rng.uniform(0.05, 0.3)), (float(rng.uniform(-50, 80)), float(rng.uniform(-50, 80))),
                          fast_axis=(math.cos(ang), math.sin(ang), 0.0), slow_axis=(-math.sin(ang), math.cos(ang), 0.0))
    tf = float(rng.uniform(0.1, 2.0))
    want, _ = oracle.background(_bg_descriptor(prof, panel, beam, tf), "f64")
    got = PixelBuffer.zeros(panel.dims, "f64")
    add_background(prof, panel, beam, tf, got)
    np.testing.assert_allclose(got.data, want, rtol=1e-12, atol=1e-300)
    got32 = PixelBuffer.zeros(panel.dims, "f32")
    add_background(prof, panel, beam, tf, got32)
    want32 = want.astype(np.float32)
    assert np.all(np.abs(got32.data.view(np.int32).astype(np.int64) - want32.view(np.int32)) <= 1)


def test_simulate_image_reference_signature_matches_reference_run(gpu):
    """simulate_image(config, image_seed) -- the reference's own call (scheduler.py:156-183) --
    with a SimulationConfig-shaped object built from this package's types, against the
    reference's accumulators for three seeds (tests/golden/sim_config.npz, made by running
    xtrace.scheduler.simulate_image on test_scheduler.py's small config): per pixel within
    one f32 ulp of each staged term."""
    import dataclasses

    from paper_2205_07976_b200 import (BeamSpectrum, CrystalModel, DetectorPanel, Executor, Orientation,
                                       StructureFactorTable, UnitCell, generate_mosaic_rotations)

    @dataclasses.dataclass
    class Config:  # the fields and crystal_for_seed of xtrace.io.SimulationConfig (io.py:122-157)
        cell: UnitCell
        n_cells: tuple
        panel: DetectorPanel
        spectrum: BeamSpectrum
        sf_table: StructureFactorTable
        background: BackgroundProfile
        mosaic_domains: int = 1
        mosaic_spread_deg: float = 0.0
        oversample: int = 1
        thickness_factor: float = 1.0

        def crystal_for_seed(self, seed):
            mosaic = generate_mosaic_rotations(seed, self.mosaic_spread_deg, self.mosaic_domains)
            return CrystalModel(cell=self.cell, orientation=Orientation(), n_cells=self.n_cells, mosaic=mosaic,
                                sf_table=self.sf_table)

    case = np.load(parity.GOLDEN / "sim_config.npz")
    config = Config(cell=UnitCell(100.0, 100.0, 100.0, 90.0, 90.0, 90.0), n_cells=(5, 5, 5),
                    panel=DetectorPanel(48, 48, 100e-6, 0.1, (23.5, 23.5)),
                    spectrum=BeamSpectrum(samples=((1.0, 1.0),), fluence=1e24,
                                          polarization_on=bool(case["polarization_on"])),
                    sf_table=StructureFactorTable({}, default_f=100.0),
                    background=BackgroundProfile(points=((0.0, 2.57), (0.07, 2.8), (0.3, 6.5))),
                    mosaic_domains=2, mosaic_spread_deg=0.05)
    with Executor.workers(2) as ex:
        for seed, want in zip(case["seeds"], case["ref_images"]):
            got = simulate_image(config, int(seed), ex)
            assert got.precision == "f64" and got.dims == (48, 48)
            np.testing.assert_allclose(got.data, want, rtol=2.0 ** -22, atol=0)
        assert ex.timing_log and ex.timing_log[-1].label == "simulate_image"


def test_fused_background_ignores_context_r_e_sqr(gpu):
    """the reference's add_background scales by the module constant R_E_SQR
    (kernels.py:44,299) whatever the spot context's r_e_sqr; simulate_image's fused launch
    composes f64(f32(spots with ctx.r_e_sqr)) + f64(f32(background with R_E_SQR))."""
    import dataclasses

    from paper_2205_07976_b200 import R_E_SQR

    water = BackgroundProfile(points=((0.0, 2.57), (0.0365, 2.58), (0.07, 2.8), (0.12, 5.0), (0.3, 6.5)))
    panel = synthetic.roi(synthetic.rayonix_panel(), 1880, 1880, 24, 32)
    ctx = dataclasses.replace(synthetic.ls49_context(panel=panel, n_channels=6, n_domains=2, compute="fp64"),
                              r_e_sqr=2.5 * R_E_SQR)
    got = simulate_image(ctx, background=water, thickness_factor=0.7)
    spots = PixelBuffer.zeros(panel.dims, "f32")
    nanobragg_spots(ctx, spots)
    bg = PixelBuffer.zeros(panel.dims, "f32")
    add_background(water, panel, ctx.spectrum, 0.7, bg)
    want = spots.data.astype(np.float64) + bg.data.astype(np.float64)
    np.testing.assert_allclose(got.data, want, rtol=2.0 ** -22, atol=0)
