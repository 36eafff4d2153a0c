"""GPU parity: the sm_100a spot kernel through the C ABI vs the reference's outputs and the oracle.

Tolerances (BASELINE.json north_star): FP64 path 1e-9 relative
on total and per-spot intensity; FP32 path 1e-4.  Extensions without a
reference (thickness, shapes, phi, multi-panel, channel shards) are checked
against the CPU oracle (oracle/) at the FP64 tolerance.
"""

import numpy as np
import pytest

import parity
from oracle import oracle
from paper_2205_07976_b200 import (
    kernel_timer,
    R_E_SQR,
    BeamSpectrum,
    Detector,
    DetectorPanel,
    Executor,
    NumericalFault,
    PatternFault,
    PhiScan,
    PixelBuffer,
    ShapeMismatchError,
    SpotsContext,
    SpotsPlan,
    add_array,
    add_noise,
    describe,
    nanobragg_spots,
    pixel_lab_position,
    solid_angle,
    synthetic,
)

pytestmark = pytest.mark.gpu

CASES = ["thomson", "scalar_match", "triclinic_pol_2wl", "pipeline_spots", "c1_toy", "tilted", "ls49_centre",
         "ls49_edge"]
FP64_TOL = 1e-9
FP32_TOL = 1e-4


def run(ctx, precision="f32"):
    out = PixelBuffer.zeros(ctx.panel.dims, precision)
    nanobragg_spots(ctx, out)
    return out


def dims(case):
    return (int(case["panel"][0]), int(case["panel"][1]))


@pytest.mark.parametrize("name", CASES)
def test_fp64_path_matches_reference(gpu, name):
    case = parity.load(name)
    got = run(parity.context(case, "fp64"), "f64").data
    m = parity.metrics(got, case["ref_f64"], dims(case))
    assert m["total"] < FP64_TOL and m["spot"] < FP64_TOL, m
    assert m["pix_abs_over_max"] < FP64_TOL, m
    # the drop-in f32 store matches the reference's store to the last ulp
    f32 = run(parity.context(case, "fp64"), "f32").data
    rel = np.abs(f32.astype(np.float64) - case["ref_f32"]) / np.maximum(np.abs(case["ref_f32"]), 1e-300)
    assert rel.max() <= 2.0 ** -23, rel.max()


@pytest.mark.parametrize("name", CASES)
def test_fp32_path_matches_reference(gpu, name):
    case = parity.load(name)
    got = run(parity.context(case, "fp32"), "f32").data
    m = parity.metrics(got, case["ref_f64"], dims(case))
    assert m["total"] < FP32_TOL and m["spot"] < FP32_TOL, m


@pytest.mark.parametrize("numerator", ["mufu", "poly"])
@pytest.mark.parametrize("name", ["c1_toy", "triclinic_pol_2wl", "ls49_centre"])
def test_fp32_numerator_variants_match_reference(gpu, monkeypatch, name, numerator):
    """Both FP32 numerators (MUFU.SIN on the XU pipe / degree-3 polynomial) on any input,
    whichever the plan would pick by samples per pixel (nbx_runtime.cu:build_plan)."""
    monkeypatch.setenv("NBX_FP32_NUM", numerator)
    case = parity.load(name)
    got = run(parity.context(case, "fp32"), "f32").data
    m = parity.metrics(got, case["ref_f64"], dims(case))
    assert m["total"] < FP32_TOL and m["spot"] < FP32_TOL, m


# ---- the reference's own kernel tests, pointed at this implementation (test_kernels.py:99-246) ----

def small_panel():
    return DetectorPanel(4, 4, 100e-6, 0.1, (1.5, 1.5))


def make(**kw):
    from paper_2205_07976_b200 import CrystalModel, MosaicDomainSet, Orientation, StructureFactorTable, UnitCell

    return CrystalModel(UnitCell(100, 100, 100, 90, 90, 90), kw.get("orientation", Orientation()),
                        kw.get("n_cells", (5, 5, 5)), kw.get("mosaic", MosaicDomainSet(np.eye(3)[None])),
                        StructureFactorTable(kw.get("entries", {}), kw.get("default_f", 100.0)))


@pytest.mark.parametrize("compute", ["fp64", "fp32"])
def test_unit_crystal_is_thomson_image(gpu, compute):
    beam = BeamSpectrum(samples=((1.0, 1.0),), fluence=1e24)
    ctx = SpotsContext(make(n_cells=(1, 1, 1)), small_panel(), beam, compute=compute)
    img = run(ctx).as_image()
    for s in range(4):
        for f in range(4):
            pos = pixel_lab_position(small_panel(), s, f, 0.5, 0.5)
            assert img[s, f] == pytest.approx(R_E_SQR * 1e24 * 100.0 ** 2 * solid_angle(small_panel(), pos),
                                              rel=1e-6)


def test_zero_fluence(gpu):
    ctx = SpotsContext(make(), small_panel(), BeamSpectrum(samples=((1.0, 1.0),), fluence=0.0))
    assert np.all(run(ctx).data == 0.0)


@pytest.mark.parametrize("compute", ["fp64", "fp32"])
def test_fluence_linear_default_f_quadratic(gpu, compute):
    def go(fluence, default_f):
        ctx = SpotsContext(make(default_f=default_f), small_panel(),
                           BeamSpectrum(samples=((1.0, 1.0),), fluence=fluence), oversample=2, compute=compute)
        return run(ctx).data.astype(np.float64)

    base = go(1e20, 50.0)
    assert np.array_equal(go(2e20, 50.0), 2.0 * base)
    assert np.array_equal(go(1e20, 100.0), 4.0 * base)
    assert (np.abs(go(3e20, 50.0) - 3.0 * base) / (3.0 * base)).max() < 1e-7


def test_dimension_mismatch(gpu):
    ctx = SpotsContext(make(), small_panel(), BeamSpectrum(samples=((1.0, 1.0),), fluence=1e24))
    with pytest.raises(ShapeMismatchError):
        nanobragg_spots(ctx, PixelBuffer.zeros((3, 4)))


@pytest.mark.parametrize("compute", ["fp64", "fp32"])
def test_numerical_fault_names_lowest_pixel(gpu, compute):
    ctx = SpotsContext(make(default_f=1e30), small_panel(), BeamSpectrum(samples=((1.0, 1.0),), fluence=1e300),
                       compute=compute)
    with pytest.raises(PatternFault) as info:
        nanobragg_spots(ctx, PixelBuffer.zeros((4, 4)))
    assert info.value.label == "nanobragg_spots"
    assert isinstance(info.value.cause, NumericalFault)
    assert info.value.index == info.value.cause.pixel == 0  # every pixel overflows; lowest is 0


def test_fault_index_is_lowest_bad_pixel(gpu):
    # only the brightest pixels overflow f32: compare with the oracle's lowest bad index
    case = parity.load("c1_toy")
    ctx = parity.context(case)
    desc = describe(ctx)
    desc.c.fluence = 1e65
    _, want = oracle.spots(desc, "f32")
    assert want > 0
    import dataclasses

    hot = dataclasses.replace(ctx, spectrum=BeamSpectrum(samples=ctx.spectrum.samples, fluence=1e65,
                                                         polarization_on=True))
    with pytest.raises(PatternFault) as info:
        nanobragg_spots(hot, PixelBuffer.zeros(ctx.panel.dims))
    assert info.value.index == want


def test_determinism_and_executor_equivalence(gpu):
    panel = DetectorPanel(80, 80, 100e-6, 0.12, (39.5, 39.5))
    beam = BeamSpectrum(samples=((1.0, 0.6), (1.01, 0.4)), fluence=1e24, polarization_on=True)
    from conftest_helpers import two_domain_mosaic

    ctx = SpotsContext(make(mosaic=two_domain_mosaic()), panel, beam, oversample=2)
    base = run(ctx).data
    for n in (1, 2, 4, 8):
        with Executor.workers(n) as ex:
            out = PixelBuffer.zeros(panel.dims)
            nanobragg_spots(ctx, out, executor=ex)
            assert np.array_equal(out.data, base)
            # like the reference's body, the call logs nothing itself; kernel_timer logs it once
            assert ex.timing_log == []
            kernel_timer(ex, "nanobragg_spots", lambda: nanobragg_spots(ctx, out, executor=ex))
            assert [r.label for r in ex.timing_log] == ["nanobragg_spots"]


# ---- extensions (no reference): GPU vs the CPU oracle ----

def oracle_check(ctx, tol=FP64_TOL):
    desc = describe(ctx)
    want, _ = oracle.spots(desc, "f64")
    got = run(ctx, "f64").data
    m = parity.metrics(got, want, ctx.panel.dims)
    assert m["total"] < tol and m["spot"] < tol, m
    return got, want


def roi_ctx(compute="fp64", centre=False, **kw):
    # off-axis ROI (sincg side lobes everywhere) or one through the direct beam (F000 spot at q = 0)
    r0, c0 = (1900, 1896) if centre else (700, 900)
    panel = synthetic.roi(synthetic.rayonix_panel(), r0, c0, 24, 40)
    return synthetic.ls49_context(panel=panel, n_channels=8, n_domains=3, compute=compute, **kw)


@pytest.mark.parametrize("shape", ["gauss", "round", "tophat"])
def test_shape_transforms_vs_oracle(gpu, shape):
    import dataclasses

    ctx = dataclasses.replace(roi_ctx(centre=True), shape=shape)
    got, want = oracle_check(ctx)
    assert want.max() > 0
    got32 = run(dataclasses.replace(ctx, compute="fp32")).data
    want, _ = oracle.spots(describe(ctx), "f64")
    m = parity.metrics(got32, want, ctx.panel.dims)
    assert m["total"] < FP32_TOL, m


def test_thickness_layers_vs_oracle(gpu):
    import dataclasses

    base = roi_ctx()
    p = base.panel
    thick = dataclasses.replace(p, thickness=320e-6, thick_steps=3, attenuation_length=60e-6)
    oracle_check(dataclasses.replace(base, panel=thick, oversample=2))


def test_thin_sensor_is_reference(gpu):
    import dataclasses

    base = roi_ctx()
    p1 = dataclasses.replace(base.panel, thick_steps=4)  # thickness 0: steps ignored
    assert np.array_equal(run(base).data, run(dataclasses.replace(base, panel=p1)).data)


def test_phi_scan_vs_oracle_and_identity(gpu):
    import dataclasses

    base = roi_ctx()
    ident = dataclasses.replace(base, phi=PhiScan(0.0, 0.0, 1))
    assert np.array_equal(run(base).data, run(ident).data)
    oracle_check(dataclasses.replace(base, phi=PhiScan(10.0, 0.3, 3, (0.0, 1.0, 0.0))))


def test_multi_panel_equals_single_panels(gpu):
    import dataclasses

    det = synthetic.jungfrau_detector(n_side=2, size=16, thickness=0.0)
    ctx = synthetic.ls49_context(panel=det, n_channels=4, n_domains=2, compute="fp64")
    got, _ = oracle_check(ctx)
    stacked = got.reshape(4, 16, 16)
    for i, p in enumerate(det.panels):
        single = run(dataclasses.replace(ctx, panel=p), "f64").data.reshape(16, 16)
        assert np.array_equal(single, stacked[i])


@pytest.mark.parametrize("compute", ["fp64", "fp32"])
def test_channel_shards_reduce_to_whole(gpu, monkeypatch, compute):
    from paper_2205_07976_b200 import _native as N

    monkeypatch.setenv("NBX_FP64_REC", "0")  # same (direct) kernel for the shards and the whole
    ctx = roi_ctx(compute)
    whole = run(ctx, "f64").data
    plan_all = SpotsPlan(ctx)
    raw = np.zeros(whole.size)
    for lo, hi in ((0, 3), (3, 8)):  # shards have their own FP32 range scales; RAW partials are scale-free
        SpotsPlan(ctx, src_begin=lo, src_end=hi, norm=0.0).run(raw, mode=N.OUT_RAW_F64)
    # FP32: shards anchor their channel chunks differently (per-pixel phase rounding ~1e-5)
    np.testing.assert_allclose(raw * plan_all.scale, whole, rtol=1e-13 if compute == "fp64" else 1e-4, atol=0)


@pytest.mark.parametrize("seed", [0, 1])
def test_fp64_channel_recurrence_matches_direct_kernel(gpu, monkeypatch, seed):
    """The FP64 channel recurrence (uniform 1/lambda runs, nbx_kernels.cu:domain_sum_f64_rec)
    against the direct per-channel FP64 kernel on an LS49 ROI through the direct beam and
    one at high resolution: 100 channels x 50 domains, per-pixel within 1e-10 of the image
    maximum, total and every spot within 1e-11."""
    from paper_2205_07976_b200 import _native as N

    for r0 in (1888, 40):
        panel = synthetic.roi(synthetic.rayonix_panel(), r0, r0, 64, 64)
        ctx = synthetic.ls49_context(synthetic.SEED + seed, panel=panel, compute="fp64")
        rec_plan = SpotsPlan(ctx)
        assert rec_plan.info.channel_runs >= 1
        rec = np.zeros(rec_plan.n_pixels)
        rec_plan.run(rec, mode=N.OUT_F64)
        monkeypatch.setenv("NBX_FP64_REC", "0")
        direct_plan = SpotsPlan(ctx)
        assert direct_plan.info.channel_runs == 0
        direct = np.zeros(direct_plan.n_pixels)
        direct_plan.run(direct, mode=N.OUT_F64)
        monkeypatch.delenv("NBX_FP64_REC")
        m = parity.metrics(rec, direct, panel.dims)
        assert m["total"] < 1e-11 and m["spot"] < 1e-11, m
        assert m["pix_abs_over_max"] < 1e-10, m


def test_fp64_recurrence_multiple_runs_matches_direct_kernel(gpu, monkeypatch):
    """Three uniform segments of different spacing plus a 300-channel segment (runs are
    capped at 128): several runs per domain, ragged run ends, unsorted input order."""
    from paper_2205_07976_b200 import _native as N

    e = np.concatenate([7000.0 + 0.7 * np.arange(37), 7050.0 + 1.3 * np.arange(50), 7140.0 + 0.25 * np.arange(13),
                        7200.0 + 0.05 * np.arange(300)])
    rng = np.random.default_rng(11)
    rng.shuffle(e)
    w = rng.uniform(0.5, 1.5, e.size)
    spec = BeamSpectrum(samples=tuple(zip((12398.419843 / e).tolist(), w.tolist())), fluence=1e24,
                        polarization_on=True)
    import dataclasses

    panel = synthetic.roi(synthetic.rayonix_panel(), 1890, 1890, 24, 24)
    ctx = dataclasses.replace(synthetic.ls49_context(panel=panel, n_domains=3, compute="fp64"), spectrum=spec)
    plan = SpotsPlan(ctx)
    assert plan.info.channel_runs >= 6
    rec = np.zeros(plan.n_pixels)
    plan.run(rec, mode=N.OUT_F64)
    monkeypatch.setenv("NBX_FP64_REC", "0")
    direct = np.zeros(plan.n_pixels)
    SpotsPlan(ctx).run(direct, mode=N.OUT_F64)
    m = parity.metrics(rec, direct, panel.dims)
    assert m["total"] < 1e-11 and m["spot"] < 1e-11 and m["pix_abs_over_max"] < 1e-10, m


def test_nonuniform_spectrum_uses_direct_fp64_kernel(gpu):
    rng = np.random.default_rng(7)
    wl = np.sort(rng.uniform(1.70, 1.76, 12))
    spec = BeamSpectrum(samples=tuple((float(w), 1.0) for w in wl), fluence=1e24)
    panel = synthetic.roi(synthetic.rayonix_panel(), 1888, 1888, 16, 16)
    ctx = synthetic.ls49_context(panel=panel, n_domains=2, compute="fp64")
    import dataclasses

    ctx = dataclasses.replace(ctx, spectrum=spec)
    assert SpotsPlan(ctx).info.channel_runs == 0
    got, _ = oracle_check(ctx)


def test_plan_runs_into_device_memory(gpu):
    import torch

    from paper_2205_07976_b200 import _native as N

    ctx = roi_ctx("fp32")
    plan = SpotsPlan(ctx)
    dev = torch.zeros(plan.n_pixels, dtype=torch.float32, device="cuda")
    torch.cuda.synchronize()
    plan.run(dev.data_ptr(), mode=N.OUT_F32, on_device=True)
    host = np.zeros(plan.n_pixels, dtype=np.float32)
    plan.run(host)
    assert np.array_equal(dev.cpu().numpy(), host)
    assert plan.kernel_ms > 0


@pytest.mark.parametrize("layout", ["single", "panels"])
@pytest.mark.parametrize("compute", ["fp64", "fp32"])
def test_pipelined_host_download_is_bitwise_the_device_image(gpu, layout, compute):
    """Host-output runs of >= 2^20 pixels are computed in row bands on two streams with the
    download of each band overlapping later bands (nbx_runtime.cu:run_plan); every pixel must
    equal the single-launch device-output image bit for bit, ragged last band included."""
    import torch

    from paper_2205_07976_b200 import _native as N

    if layout == "single":  # 1030 rows: the last of 8 bands is ragged (1030 = 7 x 136 + 78)
        panel = synthetic.roi(synthetic.rayonix_panel(), 1400, 1400, 1030, 1024)
    else:  # 20 uniform panels of 254 x 254 (Jungfrau-like): 2-D band copies across panels
        panel = synthetic.jungfrau_detector(n_side=5, size=254, thickness=0.0)
        panel = Detector(panel.panels[:20])
    ctx = synthetic.ls49_context(panel=panel, n_channels=3, n_domains=2, compute=compute)
    plan = SpotsPlan(ctx)
    assert plan.n_pixels >= 1 << 20
    for mode, dt, tdt in ((N.OUT_F32, np.float32, torch.float32), (N.OUT_F64, np.float64, torch.float64)):
        dev = torch.zeros(plan.n_pixels, dtype=tdt, device="cuda")
        torch.cuda.synchronize()
        plan.run(dev.data_ptr(), mode=mode, on_device=True)
        host = np.full(plan.n_pixels, np.nan, dtype=dt)
        plan.run(host, mode=mode)
        assert np.array_equal(dev.cpu().numpy(), host)
    plan.close()


@pytest.mark.parametrize("compute", ["fp32", "fp64"])
def test_reused_plan_tracks_table_changes(gpu, compute):
    """nanobragg_spots re-uses one plan and keeps the device F^2 grid when the structure-factor
    table is unchanged (nbx_runtime.cu: TableKey); alternating tables, a changed default_f and
    a rescaling weight must each give exactly the image of a fresh plan."""
    import dataclasses

    from paper_2205_07976_b200 import StructureFactorTable, _native as N

    base = roi_ctx(compute, centre=True)
    t0 = base.crystal.sf_table
    hkl, amp = t0.arrays()
    t1 = StructureFactorTable({tuple(int(v) for v in h): 2.0 * float(a) for h, a in zip(hkl, amp)}, t0.default_f)
    t2 = StructureFactorTable({tuple(int(v) for v in h): float(a) for h, a in zip(hkl, amp)}, t0.default_f + 3.0)
    spec_big = BeamSpectrum(samples=tuple((float(l), 1e6 * float(w)) for l, w in base.spectrum.samples),
                            fluence=base.spectrum.fluence, polarization_on=base.spectrum.polarization_on)
    ctxs = [base, dataclasses.replace(base, crystal=dataclasses.replace(base.crystal, sf_table=t1)), base,
            dataclasses.replace(base, crystal=dataclasses.replace(base.crystal, sf_table=t2)),
            dataclasses.replace(base, spectrum=spec_big), base]
    for ctx in ctxs:
        got = run(ctx, "f64").data
        fresh = np.zeros(got.size)
        SpotsPlan(ctx).run(fresh, mode=N.OUT_F64)
        assert np.array_equal(got, fresh)


@pytest.mark.parametrize("name", ["scalar_match", "triclinic_pol_2wl", "c1_toy", "ls49_centre", "ls49_edge"])
def test_sparse_fhkl_table_matches_reference(gpu, monkeypatch, name):
    """The sparse (hash) Fhkl table -- used when the reachable Miller box exceeds the dense
    grid limit -- forced on the reference fixtures: FP64 bit-identical to the dense grid (same
    F^2 values, same lookups), both paths within their tolerances of the reference."""
    monkeypatch.setenv("NBX_FHKL_HASH", "1")
    case = parity.load(name)
    plan = SpotsPlan(parity.context(case, "fp64"))
    assert plan.info.table_kind == 2
    got64 = run(parity.context(case, "fp64"), "f64").data
    m = parity.metrics(got64, case["ref_f64"], dims(case))
    assert m["total"] < FP64_TOL and m["spot"] < FP64_TOL and m["pix_abs_over_max"] < FP64_TOL, m
    got32 = run(parity.context(case, "fp32"), "f32").data
    m = parity.metrics(got32, case["ref_f64"], dims(case))
    assert m["total"] < FP32_TOL and m["spot"] < FP32_TOL, m
    monkeypatch.delenv("NBX_FHKL_HASH")
    assert np.array_equal(got64, run(parity.context(case, "fp64"), "f64").data)


@pytest.mark.parametrize("compute", ["fp64", "fp32"])
def test_virus_sized_cell_uses_sparse_table(gpu, compute):
    """A 900 A cubic cell reaches |h| ~ 600 on the C2 detector corner: a dense box of ~2e9
    cells.  The plan switches to the sparse table instead of failing; checked against the
    CPU oracle (searchsorted lookup, any index) on a high-resolution ROI."""
    import dataclasses

    from paper_2205_07976_b200 import CrystalModel, MosaicDomainSet, StructureFactorTable, UnitCell

    rng = np.random.default_rng(3)
    hkl = rng.integers(-400, 401, size=(20000, 3))
    entries = {tuple(int(v) for v in h): float(a) for h, a in zip(hkl, rng.uniform(10, 300, len(hkl)))}
    panel = synthetic.roi(synthetic.rayonix_panel(), 60, 200, 12, 16)
    base = synthetic.ls49_context(panel=panel, n_channels=3, n_domains=2, compute=compute)
    crystal = CrystalModel(UnitCell(900, 900, 900, 90, 90, 90), base.crystal.orientation, (5, 5, 5),
                           MosaicDomainSet(base.crystal.mosaic.rotations), StructureFactorTable(entries, 1.0))
    ctx = dataclasses.replace(base, crystal=crystal)
    plan = SpotsPlan(ctx)
    assert plan.info.table_kind == 2
    oracle_check(ctx, FP64_TOL if compute == "fp64" else FP32_TOL)


@pytest.mark.parametrize("compute", ["fp64", "fp32"])
def test_long_spectrum_is_channel_sharded_on_one_device(gpu, compute):
    """20,000 wavelength samples (the reference has no limit; one launch holds 8192): the call
    splits the spectrum into channel shards with the global normalisation, accumulates FP64
    partials and scales once -- checked against the oracle, and the f32 store within 1 ulp of
    the f64 one."""
    import dataclasses

    e = 6500.0 + 0.1 * np.arange(20000)
    rng = np.random.default_rng(2)
    spec = BeamSpectrum(samples=tuple(zip((12398.419843 / e).tolist(), rng.uniform(0.2, 1.0, e.size).tolist())),
                        fluence=1e24, polarization_on=True)
    panel = synthetic.roi(synthetic.rayonix_panel(), 1880, 1890, 10, 12)
    ctx = dataclasses.replace(synthetic.ls49_context(panel=panel, n_domains=1, compute=compute), spectrum=spec)
    got, _ = oracle_check(ctx, FP64_TOL if compute == "fp64" else FP32_TOL)
    f32 = run(ctx, "f32").data
    np.testing.assert_allclose(f32, got, rtol=2.0 ** -23, atol=0)
    # a resident plan holds at most 8192 sources: a clear argument error, not a
    # launch failure; its shards are fine
    with pytest.raises(ValueError, match="max 8192"):
        SpotsPlan(ctx)
    SpotsPlan(ctx, src_begin=0, src_end=8192).close()
    # simulate_image / run_campaign on the long spectrum: the accumulator composed stage by
    # stage equals f64(f32(spots)) + f64(f32(background)) bit for bit, and the campaign's
    # .bin payload is that accumulator rounded to f32
    import tempfile

    from paper_2205_07976_b200 import BackgroundProfile, add_background, simulate_image
    from paper_2205_07976_b200.io import read_image, run_campaign

    water = BackgroundProfile(points=((0.0, 2.57), (0.07, 2.8), (0.12, 5.0), (0.3, 6.5)))
    img = simulate_image(ctx, background=water, thickness_factor=0.8)
    bg = PixelBuffer.zeros(panel.dims, "f32")
    add_background(water, panel, spec, 0.8, bg)
    want = f32.astype(np.float64) + bg.data.astype(np.float64)
    assert np.array_equal(img.data, want)
    with tempfile.TemporaryDirectory() as d:
        res = run_campaign(lambda i: ctx, 2, d, background=water, thickness_factor=0.8)
        for path in res.paths:
            assert np.array_equal(read_image(path)[0].reshape(-1), want.astype(np.float32))


def test_pipelined_image_mode_with_background_is_bitwise_the_device_image(gpu):
    """simulate_image's fused spots + background accumulator (NBX_OUT_IMAGE_F64) through the
    banded host download equals the single-launch device-output image bit for bit."""
    import torch

    from paper_2205_07976_b200 import BackgroundProfile, _native as N

    water = BackgroundProfile(points=((0.0, 2.57), (0.0365, 2.58), (0.07, 2.8), (0.12, 5.0), (0.3, 6.5)))
    panel = synthetic.roi(synthetic.rayonix_panel(), 1400, 1400, 1030, 1024)
    ctx = synthetic.ls49_context(panel=panel, n_channels=3, n_domains=2, compute="fp32")
    desc = describe(ctx, background=water, thickness_factor=0.8)
    cx = N.context()
    dev = torch.zeros(panel.n_pixels, dtype=torch.float64, device="cuda")
    torch.cuda.synchronize()
    bad = N.C.c_int64(-1)
    assert cx.lib.nbx_spots(cx.handle, N.C.byref(desc.c), 1, N.OUT_IMAGE_F64, dev.data_ptr(), 1, N.C.byref(bad)) == 0
    host = np.full(panel.n_pixels, np.nan)
    assert cx.lib.nbx_spots(cx.handle, N.C.byref(desc.c), 1, N.OUT_IMAGE_F64, host.ctypes.data, 0,
                            N.C.byref(bad)) == 0
    assert np.array_equal(dev.cpu().numpy(), host)


def test_add_array_upcast_semantics(gpu):
    lhs = PixelBuffer((1, 3), "f64", [0.0, 1.0, 2.0])
    rhs = PixelBuffer((1, 3), "f32", [0.1, 0.5, 0.25])
    add_array(lhs, rhs)
    assert lhs.data.tolist() == [0.10000000149011612, 1.5, 2.25]


def test_poisson_noise_bit_exact_with_host_twin(gpu):
    rng = np.random.default_rng(11)
    mean = np.concatenate([rng.uniform(0, 12, 50000), rng.uniform(12, 1e4, 50000), [0.0, 1e7]])
    for prec in ("f64", "f32"):
        buf = PixelBuffer((1, mean.size), prec, mean)
        dev = add_noise(buf, seed=1234, image=7).data
        host = oracle.poisson(buf.data, 1234, 7)
        assert np.array_equal(dev, host), prec
    # statistics sanity: mean and variance of a constant field
    flat = PixelBuffer((1, 200000), "f64", np.full(200000, 37.5))
    draws = add_noise(flat, seed=9).data
    assert abs(draws.mean() - 37.5) < 0.1 and abs(draws.var() - 37.5) < 1.0


@pytest.mark.parametrize("compute", ["fp64", "fp32"])
def test_channel_sharded_path_single_rank(gpu, compute):
    """The C5 path (raw FP64 partial -> reduce -> nbx_finalize) on one rank equals the direct
    image (FP32 is the C5 bench's path: its partials must not carry the FP32 range scale)."""
    from paper_2205_07976_b200 import parallel

    ctx = roi_ctx(compute)
    rtol = 1e-13 if compute == "fp64" else 2e-6
    direct = run(ctx, "f64").data
    # the partial -> finalize pieces themselves (a single rank's default call skips them: one
    # shard is the whole spectrum, so it takes the single-image call with the banded download)
    pieces = dict(partial=parallel._gpu_partial, finalize=parallel._gpu_finalize)
    got = parallel.simulate_channel_sharded(ctx, PixelBuffer.zeros(ctx.panel.dims, "f64"), **pieces)
    np.testing.assert_allclose(got.data, direct, rtol=rtol, atol=0)
    f32 = parallel.simulate_channel_sharded(ctx, **pieces)
    assert f32.precision == "f32"
    np.testing.assert_allclose(f32.data, direct.astype(np.float32), rtol=max(rtol, 2e-7))
    default = parallel.simulate_channel_sharded(ctx)  # single rank: the single-image call
    assert default.precision == "f32" and np.array_equal(default.data, run(ctx, "f32").data)


def test_nanobragg_facade_matches_api(gpu):
    from paper_2205_07976_b200 import nanoBragg, shapetype

    sim = nanoBragg(detpixels_slowfast=(48, 40), pixel_size_mm=0.1, Ncells_abc=(5, 6, 7), oversample=2)
    sim.distance_mm = 90.0
    sim.wavelength_A = 1.1
    sim.unit_cell_tuple = (60, 70, 80, 90, 95, 90)
    sim.mosaic_spread_deg, sim.mosaic_domains, sim.mosaic_seed = 0.1, 3, 5
    sim.Fhkl_tuple = ([(1, 0, 0), (0, 1, 1)], [200.0, 90.0])
    sim.default_F = 10.0
    sim.add_nanoBragg_spots()
    want = run(sim.to_context(), "f64").as_image()
    assert np.array_equal(sim.raw_pixels, want)
    sim.add_nanoBragg_spots()
    assert np.array_equal(sim.raw_pixels, 2 * want)
    sim.xtal_shape = shapetype.Gauss
    assert sim.to_context().shape == "gauss"
    sim.seed = 3
    before = sim.raw_pixels.copy()
    sim.add_noise()
    assert np.all(sim.raw_pixels == np.round(sim.raw_pixels)) and not np.array_equal(before, sim.raw_pixels)


def test_reference_duck_typed_context(gpu):
    """The drop-in accepts reference-shaped objects (no PhiScan / arrays() / compute fields)."""
    import types

    case = parity.load("scalar_match")
    ours = parity.context(case)
    table = types.SimpleNamespace(entries=dict(ours.crystal.sf_table.entries),
                                  default_f=ours.crystal.sf_table.default_f)
    crystal = types.SimpleNamespace(cell=ours.crystal.cell, n_cells=ours.crystal.n_cells, sf_table=table,
                                    mosaic=ours.crystal.mosaic,
                                    rotated_real_bases=lambda: ours.crystal.rotated_real_bases())
    ref_ctx = types.SimpleNamespace(crystal=crystal, panel=ours.panel, spectrum=ours.spectrum,
                                    oversample=ours.oversample, r_e_sqr=ours.r_e_sqr)
    out = types.SimpleNamespace(data=np.zeros(16, np.float32), dims=(4, 4), precision="f32")
    nanobragg_spots(ref_ctx, out)
    assert np.array_equal(out.data, run(ours).data)


def test_batch_api_equals_single_images(gpu):
    import ctypes as C

    from paper_2205_07976_b200 import _native as N

    ctxs = [roi_ctx(seed=synthetic.SEED + i) for i in range(3)]
    descs = [describe(c) for c in ctxs]
    arr = (N.SpotsDesc * 3)(*[d.c for d in descs])
    outs = [np.zeros(c.panel.n_pixels, np.float32) for c in ctxs]
    ptrs = (C.c_void_p * 3)(*[o.ctypes.data for o in outs])
    cx = N.context()
    bad = C.c_int64(-1)
    assert cx.lib.nbx_spots_batch(cx.handle, arr, 3, 0, N.OUT_F32, ptrs, 0, C.byref(bad)) == 0
    for c, o in zip(ctxs, outs):
        assert np.array_equal(o, run(c).data)


def test_concurrent_host_threads_share_one_context(gpu):
    """Python threads calling the drop-in API at once (ctypes drops the GIL) serialise on the
    context lock: every thread's images equal the same images rendered one after another."""
    from concurrent.futures import ThreadPoolExecutor

    from paper_2205_07976_b200 import image_stats, simulate_image

    panel = synthetic.roi(synthetic.rayonix_panel(), 700, 900, 48, 64)
    ctxs = [synthetic.ls49_context(synthetic.SEED + i, panel=panel, n_channels=6, n_domains=2,
                                   compute=("fp32", "fp64")[i % 2]) for i in range(8)]

    def render(c):
        a = run(c, "f32").data.copy()
        b = simulate_image(c).data.copy()
        return a, b, image_stats(PixelBuffer(c.panel.dims, "f64", b)).total

    serial = [render(c) for c in ctxs]
    with ThreadPoolExecutor(8) as pool:
        threaded = list(pool.map(render, ctxs * 3))
    for i, (a, b, t) in enumerate(threaded):
        sa, sb, st = serial[i % len(ctxs)]
        assert np.array_equal(a, sa) and np.array_equal(b, sb) and t == st


@pytest.mark.parametrize("compute", ["fp64", "fp32"])
def test_ragged_multi_panel_and_single_pixel_panels(gpu, compute):
    """Edge shapes: panels of 1, 7 and 1031 rows (ragged: not a multiple of the 8-row block
    line, one panel a single pixel row) sharing 19 columns, and a 1x1 panel -- against the
    oracle and, panel by panel, against single-panel runs (bit for bit)."""
    import dataclasses

    from paper_2205_07976_b200 import Detector

    base = synthetic.roi(synthetic.rayonix_panel(), 700, 900, 8, 19)
    panels = tuple(dataclasses.replace(base, slow_pixels=n, beam_center=(base.beam_center[0] - 40 * k,
                                                                         base.beam_center[1] + 3 * k))
                   for k, n in enumerate((1, 7, 1031)))
    det = Detector(panels)
    ctx = synthetic.ls49_context(panel=det, n_channels=5, n_domains=2, compute=compute)
    tol = FP64_TOL if compute == "fp64" else FP32_TOL
    want, _ = oracle.spots(describe(dataclasses.replace(ctx, panel=Detector(panels[:2]))), "f64")
    got = run(ctx, "f64").data
    m = parity.metrics(got[: 8 * 19], want, (8, 19))
    assert m["total"] < tol, m
    off = 0
    for p in panels:
        single = run(dataclasses.replace(ctx, panel=p), "f64").data
        assert np.array_equal(single, got[off: off + single.size])
        off += single.size
    one = dataclasses.replace(base, slow_pixels=1, fast_pixels=1)
    c1 = dataclasses.replace(ctx, panel=one)
    w1, _ = oracle.spots(describe(c1), "f64")
    g1 = run(c1, "f64").data
    assert abs(g1[0] - w1[0]) <= tol * abs(w1[0]) + 1e-300


def test_c_abi_argument_errors_leave_the_context_usable(gpu):
    """Every entry point rejects bad arguments with NBX_ERR_ARG and a message (no crash, no
    out-of-bounds write), and the context keeps working afterwards (include/nbx.h contract)."""
    from paper_2205_07976_b200 import _native as N

    cx = N.context()
    lib, h = cx.lib, cx.handle
    ctx = synthetic.c1_context()
    desc = describe(ctx)
    out = np.zeros(ctx.panel.n_pixels, np.float32)
    bad = N.C.c_int64(-1)
    dev = N.C.c_void_p()
    calls = {
        "spots NULL ctx": lambda: lib.nbx_spots(None, N.C.byref(desc.c), 0, 0, out.ctypes.data, 0, N.C.byref(bad)),
        "spots NULL desc": lambda: lib.nbx_spots(h, None, 0, 0, out.ctypes.data, 0, N.C.byref(bad)),
        "spots NULL out": lambda: lib.nbx_spots(h, N.C.byref(desc.c), 0, 0, None, 0, N.C.byref(bad)),
        "spots mode": lambda: lib.nbx_spots(h, N.C.byref(desc.c), 0, 9, out.ctypes.data, 0, N.C.byref(bad)),
        "spots compute": lambda: lib.nbx_spots(h, N.C.byref(desc.c), 7, 0, out.ctypes.data, 0, N.C.byref(bad)),
        "plan_run NULL": lambda: lib.nbx_plan_run(None, 0, out.ctypes.data, 0, N.C.byref(bad)),
        "finalize image mode": lambda: lib.nbx_finalize(h, out.ctypes.data, out.size, 1.0, N.OUT_IMAGE_F32,
                                                        out.ctypes.data, 0, N.C.byref(bad)),
        "reduce_slots raw mode": lambda: lib.nbx_reduce_slots(h, out.ctypes.data, 1, out.size, 1.0, N.OUT_RAW_F64,
                                                              out.ctypes.data, 0, N.C.byref(bad)),
        "stats empty": lambda: lib.nbx_image_stats(h, out.ctypes.data, 0, 0, 0, (N.C.c_double * 4)()),
        "noise dtype": lambda: lib.nbx_add_noise(h, out.ctypes.data, out.ctypes.data, out.size, 7, 1, 0, 0),
        "background mode": lambda: lib.nbx_background(h, N.C.byref(desc.c), N.OUT_IMAGE_F64, out.ctypes.data, 0,
                                                      N.C.byref(bad)),
        "campaign count": lambda: lib.nbx_campaign(h, N.C.byref(desc.c), -1, 0, None, None, N.C.byref(bad)),
        "ipc_open NULL": lambda: lib.nbx_ipc_open(h, None, N.C.byref(dev)),
        "ipc_alloc size": lambda: lib.nbx_ipc_alloc(h, 0, N.C.byref(dev), N.C.create_string_buffer(64)),
    }
    for name, call in calls.items():
        assert call() == N.NBX_ERR_ARG, name
        if "NULL ctx" not in name and "plan_run" not in name:
            assert cx.error(), name
    ref = run(ctx).data
    again = PixelBuffer.zeros(ctx.panel.dims)
    nanobragg_spots(ctx, again)
    assert np.array_equal(again.data, ref)


def test_grid_limits_tall_panel_and_many_panels(gpu):
    """Beyond one launch's grid (65535 block lines of 8 rows, 65535 panel slices): a 600,000-row
    panel and a 70,000-panel detector are launched in row / panel chunks -- pieces equal
    single-panel runs bit for bit."""
    import dataclasses

    from paper_2205_07976_b200 import Detector

    base = synthetic.roi(synthetic.rayonix_panel(), 1900, 1900, 8, 2)
    ctx = synthetic.ls49_context(panel=base, n_channels=2, n_domains=1, compute="fp64")
    tall = dataclasses.replace(base, slow_pixels=600_000)
    import torch

    from paper_2205_07976_b200 import _native as N

    plan = SpotsPlan(dataclasses.replace(ctx, panel=tall))  # device output: one launch request, row-chunked
    dev = torch.zeros(plan.n_pixels, dtype=torch.float64, device="cuda")
    plan.run(dev.data_ptr(), mode=N.OUT_F64, on_device=True)
    img = dev.cpu().numpy().reshape(600_000, 2)
    assert np.array_equal(img, run(dataclasses.replace(ctx, panel=tall), "f64").data.reshape(600_000, 2))
    for r0 in (0, 524_280 - 3, 599_990):
        piece = dataclasses.replace(base, slow_pixels=8, beam_center=(base.beam_center[0] - r0, base.beam_center[1]))
        want = run(dataclasses.replace(ctx, panel=piece), "f64").data.reshape(8, 2)
        assert np.array_equal(img[r0:r0 + 8], want[: min(8, 600_000 - r0)]), r0
    one = dataclasses.replace(base, slow_pixels=1, fast_pixels=1)
    panels = tuple(dataclasses.replace(one, beam_center=(base.beam_center[0] + (k % 7), base.beam_center[1]))
                   for k in range(70_000))
    many = run(dataclasses.replace(ctx, panel=Detector(panels)), "f64").data
    for k in (0, 65_534, 65_535, 69_999):
        want = run(dataclasses.replace(ctx, panel=panels[k]), "f64").data
        assert many[k] == want[0], k


def test_caller_stream_and_probe(gpu):
    """nbx_ctx_set_stream: launches go to the caller's stream (a torch stream here) with the same
    image; NULL restores the context's own stream.  nbx_ctx_synchronize and the FMA-peak probe
    the bench's roofline uses answer sensibly."""
    import torch

    from paper_2205_07976_b200 import _native as N

    cx = N.context()
    ctx = synthetic.ls49_context(panel=synthetic.roi(synthetic.rayonix_panel(), 1800, 1800, 40, 64), n_channels=8,
                                 n_domains=2, compute="fp32")
    plan = SpotsPlan(ctx)
    a = torch.zeros(plan.n_pixels, dtype=torch.float32, device="cuda")
    plan.run(a.data_ptr(), on_device=True)
    s = torch.cuda.Stream()
    b = torch.zeros_like(a)
    with cx.lock:
        assert cx.lib.nbx_ctx_set_stream(cx.handle, N.C.c_void_p(s.cuda_stream)) == N.NBX_OK
    try:
        plan.run(b.data_ptr(), on_device=True)
        s.synchronize()
        assert torch.equal(a, b)
        with cx.lock:
            assert cx.lib.nbx_ctx_synchronize(cx.handle) == N.NBX_OK
    finally:
        with cx.lock:
            assert cx.lib.nbx_ctx_set_stream(cx.handle, None) == N.NBX_OK
    plan.close()
    for fp64, floor in ((0, 20.0), (1, 10.0)):
        tf = N.C.c_double(0.0)
        with cx.lock:
            assert cx.lib.nbx_probe_fma_peak(cx.handle, fp64, N.C.byref(tf)) == N.NBX_OK
        assert floor < tf.value < 200.0, (fp64, tf.value)


@pytest.mark.parametrize("compute", ["fp64", "fp32"])
def test_vectorised_stores_any_alignment(gpu, compute):
    """The epilogue writes full 32-pixel warp rows as float4 / double2 when the row's first
    element is 16-byte aligned and falls back to scalar stores otherwise: a device output
    offset by 1..3 elements, odd panel widths and a partial last warp give the same pixels."""
    import torch

    from paper_2205_07976_b200 import _native as N

    for rows, cols in ((6, 64), (5, 70), (3, 33)):
        panel = synthetic.roi(synthetic.rayonix_panel(), 1880, 1880, rows, cols)
        ctx = synthetic.ls49_context(panel=panel, n_channels=6, n_domains=2, compute=compute)
        plan = SpotsPlan(ctx)
        for mode, dt in ((N.OUT_F32, torch.float32), (N.OUT_F64, torch.float64)):
            ref = None
            for off in range(4):
                buf = torch.zeros(plan.n_pixels + 4, dtype=dt, device="cuda")
                plan.run(buf.data_ptr() + off * buf.element_size(), mode=mode, on_device=True)
                img = buf[off:off + plan.n_pixels].cpu().numpy()
                assert np.all(buf[:off].cpu().numpy() == 0) and np.all(buf[off + plan.n_pixels:].cpu().numpy() == 0)
                if ref is None:
                    ref = img
                assert np.array_equal(img, ref), (rows, cols, mode, off)
        plan.close()
