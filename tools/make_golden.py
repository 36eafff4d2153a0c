"""Generate tests/golden/*.npz by running the REFERENCE implementation.

Run here (where /root/reference exists):  python tools/make_golden.py
The GPU box never runs this; it only reads the committed fixtures.

Each fixture stores the exact inputs as plain arrays (cell, orientation,
mosaic rotations, Fhkl entries, panel, spectrum, oversample) plus
  ref_f32 : xtrace.kernels.nanobragg_spots output (FP64 math, f32 store)
  ref_f64 : the same code with the f32 cast intercepted ("oracle64",
            SURVEY §8 C1): the FP64 values before the store
Checks done while generating: f32(ref_f64) == ref_f32 bit for bit, and the
package's own mosaic generator reproduces the reference's matrices exactly.
"""
from __future__ import annotations

import json
import sys
import time
import types
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
sys.path.insert(0, "/root/reference/pkg/src")

import xtrace.kernels as xk  # noqa: E402
import xtrace.model as xm  # noqa: E402

from paper_2205_07976_b200 import synthetic as syn  # noqa: E402

OUT = ROOT / "tests" / "golden"


def rotation_about(axis, angle_deg):
    axis = np.asarray(axis, dtype=float)
    axis = axis / np.linalg.norm(axis)
    ang = np.radians(angle_deg)
    ax, ay, az = axis
    k = np.array([[0, -az, ay], [az, 0, -ax], [-ay, ax, 0]])
    return np.eye(3) + np.sin(ang) * k + (1 - np.cos(ang)) * (k @ k)


def run_reference(case):
    """(ref_f32, ref_f64) from xtrace for one case dict of arrays."""
    cell = xm.UnitCell(*case["cell"])
    crystal = xm.CrystalModel(
        cell=cell,
        orientation=xm.Orientation(case["orientation"]),
        n_cells=tuple(int(x) for x in case["n_cells"]),
        mosaic=xm.MosaicDomainSet(case["mosaic"]),
        sf_table=xm.StructureFactorTable(
            {tuple(int(v) for v in h): float(a) for h, a in zip(case["hkl"], case["amp"])},
            default_f=float(case["default_f"])),
    )
    p = case["panel"]
    panel = xm.DetectorPanel(int(p[0]), int(p[1]), float(p[2]), float(p[3]), (float(p[4]), float(p[5])),
                             fast_axis=tuple(case["fast_axis"]), slow_axis=tuple(case["slow_axis"]))
    beam = xm.BeamSpectrum(samples=tuple(map(tuple, case["samples"])), fluence=float(case["fluence"]),
                           polarization_on=bool(case["pol"]), beam_direction=tuple(case["beam_dir"]))
    ctx = xk.SpotsContext(crystal, panel, beam, oversample=int(case["oversample"]))
    out32 = xk.PixelBuffer.zeros(panel.dims)
    xk.nanobragg_spots(ctx, out32)

    # oracle64: same code, cast intercepted (kernels.py:271-273)
    cap = np.zeros(panel.n_pixels)
    shim = types.SimpleNamespace(**{k: getattr(np, k) for k in dir(np) if not k.startswith("__")})
    shim.float32 = np.float64
    real_np, real_store = xk.np, xk._store_checked

    def store(out_slice, values, lo):
        cap[lo:lo + len(values)] = values
        real_store(out_slice, values, lo)

    xk.np, xk._store_checked = shim, store
    try:
        out64 = xk.PixelBuffer.zeros(panel.dims)
        xk.nanobragg_spots(ctx, out64)
    finally:
        xk.np, xk._store_checked = real_np, real_store
    assert np.array_equal(cap.astype(np.float32), out32.data), "f32(oracle64) != reference store"
    return out32.data.copy(), cap


def run_reference_bg(case):
    """(ref_bg_f32, ref_bg_f64) from xtrace.kernels.add_background (kernels.py:279-312)."""
    p = case["panel"]
    panel = xm.DetectorPanel(int(p[0]), int(p[1]), float(p[2]), float(p[3]), (float(p[4]), float(p[5])),
                             fast_axis=tuple(case["fast_axis"]), slow_axis=tuple(case["slow_axis"]))
    beam = xm.BeamSpectrum(samples=tuple(map(tuple, case["samples"])), fluence=float(case["fluence"]),
                           polarization_on=bool(case["pol"]), beam_direction=tuple(case["beam_dir"]))
    prof = xm.BackgroundProfile(points=tuple(map(tuple, case["bg_points"])))
    tf = float(case["thickness_factor"])
    out32 = xk.PixelBuffer.zeros(panel.dims)
    xk.add_background(prof, panel, beam, tf, out32)
    cap = np.zeros(panel.n_pixels)
    shim = types.SimpleNamespace(**{k: getattr(np, k) for k in dir(np) if not k.startswith("__")})
    shim.float32 = np.float64
    real_np, real_store = xk.np, xk._store_checked

    def store(out_slice, values, lo):
        cap[lo:lo + len(values)] = values
        real_store(out_slice, values, lo)

    xk.np, xk._store_checked = shim, store
    try:
        xk.add_background(prof, panel, beam, tf, xk.PixelBuffer.zeros(panel.dims))
    finally:
        xk.np, xk._store_checked = real_np, real_store
    assert np.array_equal(cap.astype(np.float32), out32.data)
    return out32.data.copy(), cap


def base_case(**kw):
    c = dict(cell=(100.0, 100.0, 100.0, 90.0, 90.0, 90.0), orientation=np.eye(3), n_cells=(5, 5, 5),
             mosaic=np.eye(3)[None], hkl=np.zeros((0, 3), np.int32), amp=np.zeros(0), default_f=100.0,
             panel=(4, 4, 100e-6, 0.1, 1.5, 1.5), fast_axis=(1.0, 0.0, 0.0), slow_axis=(0.0, 1.0, 0.0),
             samples=np.array([[1.0, 1.0]]), fluence=1e24, pol=False, beam_dir=(0.0, 0.0, 1.0), oversample=1)
    c.update(kw)
    return c


def two_domain():
    return np.stack([rotation_about([1, 0, 0], 0.02), rotation_about([0, 1, 1], -0.03)])


def entries(d):
    hkl = np.array(list(d.keys()), dtype=np.int32).reshape(-1, 3)
    amp = np.array(list(d.values()), dtype=float)
    return hkl, amp


def ls49_case(r0, c0, rows, cols, n_channels, n_domains, seed=syn.SEED, compute_note=""):
    crystal = syn.ls49_crystal(seed, n_domains)
    # the package's mosaic draw must equal the reference's, bit for bit
    ref_mos = xm.generate_mosaic_rotations(seed, 0.05, n_domains).rotations
    assert np.array_equal(ref_mos, crystal.mosaic.rotations), "mosaic generator differs from the reference"
    spec = syn.ls49_spectrum(n_channels, 7070.0, 1.0, seed)
    full = syn.rayonix_panel()
    hkl, amp = crystal.sf_table.arrays()
    return base_case(cell=syn.LS49_CELL, orientation=crystal.orientation.u, n_cells=syn.LS49_NCELLS,
                     mosaic=crystal.mosaic.rotations, hkl=hkl, amp=amp, default_f=0.0,
                     panel=(rows, cols, full.pixel_size, full.distance, full.beam_center[0] - r0,
                            full.beam_center[1] - c0),
                     samples=np.array(spec.samples), fluence=spec.fluence, pol=True)


CASES = {
    # test_kernels.py:100-111 -- unit crystal is the Thomson image
    "thomson": base_case(n_cells=(1, 1, 1)),
    # test_kernels.py:120-145
    "scalar_match": base_case(mosaic=two_domain(), oversample=2,
                              **dict(zip(("hkl", "amp"), entries({(0, 0, 0): 300.0, (1, 0, 0): 50.0,
                                                                  (0, 1, 0): 80.0})))),
    # test_kernels.py:147-175
    "triclinic_pol_2wl": base_case(cell=(60, 70, 80, 85, 92, 103), orientation=rotation_about([0.2, 1.0, -0.4], 13.0),
                                   n_cells=(4, 3, 6), mosaic=two_domain(), default_f=20.0, oversample=3,
                                   panel=(5, 3, 150e-6, 0.08, 2.0, 1.25),
                                   samples=np.array([[1.0, 0.75], [1.02, 0.25]]), fluence=5e23, pol=True,
                                   **dict(zip(("hkl", "amp"), entries({(1, 1, 1): 40.0})))),
    # test_kernels.py:439-471 (spot part of the pipeline)
    "pipeline_spots": base_case(mosaic=two_domain(), oversample=2, samples=np.array([[1.0, 0.6], [1.05, 0.4]]),
                                pol=True, **dict(zip(("hkl", "amp"), entries({(1, 0, 0): 250.0})))),
    # C1 toy (test_acceptance.py:52-65 shape at 256^2, bc on a pixel centre -> limit branch)
    "c1_toy": base_case(panel=(256, 256, 100e-6, 0.1, 127.5, 127.5), pol=True,
                        **dict(zip(("hkl", "amp"), entries({(1, 0, 0): 250.0})))),
    # tilted panel axes + off-axis beam
    "tilted": base_case(cell=(50, 60, 70, 90, 90, 90), orientation=rotation_about([1, 2, 3], 40.0),
                        n_cells=(7, 8, 9), panel=(24, 20, 172e-6, 0.09, 11.3, 8.7),
                        fast_axis=tuple(rotation_about([0, 1, 0], 10.0) @ [1.0, 0, 0]),
                        slow_axis=tuple(rotation_about([0, 1, 0], 10.0) @ [0, 1.0, 0]),
                        beam_dir=tuple(rotation_about([1, 0, 0], 3.0) @ [0, 0, 1.0]),
                        samples=np.array([[1.3, 0.2], [1.31, 0.5], [1.32, 0.3]]), pol=True, default_f=10.0,
                        **dict(zip(("hkl", "amp"), entries({(1, 1, 0): 30.0, (0, 1, 1): 70.0, (2, 0, 1): 5.0})))),
    # LS49-shape ROIs: one through the beam centre (q = 0 pixel, F000), one at high resolution
    "ls49_centre": ls49_case(1888, 1888, 64, 64, 20, 10),
    "ls49_edge": ls49_case(96, 160, 48, 96, 100, 50),
}


WATER = np.array([[0.0, 2.57], [0.0365, 2.58], [0.07, 2.8], [0.12, 5.0], [0.162, 8.0], [0.3, 6.5]])
BG_CASES = {
    # test_kernels.py:249-260 flat profile, polarization off
    "bg_flat": base_case(bg_points=np.array([[0.0, 3.0], [1.0, 3.0]]), thickness_factor=1.0),
    # test_kernels.py:267-279
    "bg_scalar": base_case(bg_points=np.array([[0.0, 10.0], [0.5, 2.0]]), thickness_factor=1.3, pol=True),
    # test_kernels.py:281-293 (80x80, two wavelengths, water profile)
    "bg_water_80": base_case(panel=(80, 80, 100e-6, 0.12, 39.5, 39.5), samples=np.array([[1.0, 0.7], [1.05, 0.3]]),
                             pol=True, bg_points=WATER, thickness_factor=1.0),
}


def pipeline_case():
    """test_kernels.py:439-471: spots + background -> f64 accumulator via add_array."""
    case = base_case(mosaic=two_domain(), oversample=2, samples=np.array([[1.0, 0.6], [1.05, 0.4]]), pol=True,
                     bg_points=WATER[:4], thickness_factor=1.0,
                     **dict(zip(("hkl", "amp"), entries({(1, 0, 0): 250.0}))))
    s32, _ = run_reference(case)
    b32, _ = run_reference_bg(case)
    acc = xk.PixelBuffer.zeros((4, 4), "f64")
    xk.add_array(acc, xk.PixelBuffer((4, 4), "f32", s32))
    xk.add_array(acc, xk.PixelBuffer((4, 4), "f32", b32))
    return case, acc.data.copy()


STATS_SPECS = [(15, "f32"), (8192, "f64"), (3 * 8192 + 5, "f32"), (1_000_000, "f32"), (1_000_000, "f64")]


def stats_values(n: int, precision: str) -> np.ndarray:
    """Lognormal over ~14 decades (summation order matters), seeded by n."""
    rng = np.random.default_rng(n)
    return np.exp(rng.normal(0.0, 8.0, n)).astype(np.float32 if precision == "f32" else np.float64)


def stats_case():
    """xtrace.kernels.image_stats (kernels.py:346-371) on seeded arrays: the reference's bits."""
    rows = []
    for n, prec in STATS_SPECS:
        v = stats_values(n, prec)
        st = xk.image_stats(xk.PixelBuffer((1, n), prec, v))
        rows.append([st.min, st.max, st.mean, st.total])
    return {"n": np.array([n for n, _ in STATS_SPECS]), "precision": np.array([p for _, p in STATS_SPECS]),
            "ref_stats": np.array(rows)}


SIM_SEEDS = (11, 12, 13)


def sim_config_case():
    """xtrace.scheduler.simulate_image(config, image_seed) (scheduler.py:156-183) on the
    reference's own small scheduler config (test_scheduler.py:30-45): the f64 accumulator of
    spots + background for three image seeds (each seed draws its own mosaic domains)."""
    import xtrace.io as xio
    import xtrace.scheduler as xs

    config = xio.SimulationConfig(
        cell=xm.UnitCell(100.0, 100.0, 100.0, 90.0, 90.0, 90.0), n_cells=(5, 5, 5),
        panel=xm.DetectorPanel(48, 48, 100e-6, 0.1, (23.5, 23.5)),
        spectrum=xm.BeamSpectrum(samples=((1.0, 1.0),), fluence=1e24),
        sf_table=xm.StructureFactorTable({}, default_f=100.0),
        background=xm.BackgroundProfile(points=((0.0, 2.57), (0.07, 2.8), (0.3, 6.5))),
        mosaic_domains=2, mosaic_spread_deg=0.05, oversample=1, seed=0)
    images = np.stack([xs.simulate_image(config, s).data.copy() for s in SIM_SEEDS])
    return {"seeds": np.array(SIM_SEEDS), "ref_images": images, "polarization_on": config.spectrum.polarization_on}


def image_io_case():
    """xtrace.io.write_image (io.py:403-434) on a seeded f64 accumulator with panel, spectrum,
    seed and index: the exact .bin bytes and .json text the reference writes."""
    import tempfile

    import xtrace.io as xio

    rng = np.random.default_rng(7)
    data = rng.lognormal(0.0, 3.0, 24 * 40)
    panel = xm.DetectorPanel(24, 40, 88.6e-6, 0.1417, (11.5, 19.5))
    spectrum = xm.BeamSpectrum(samples=((1.7, 0.5), (1.71, 0.25), (1.72, 0.25)), fluence=1e24)
    with tempfile.TemporaryDirectory() as d:
        path = xio.write_image(xk.PixelBuffer((24, 40), "f64", data), Path(d) / "img_000007", panel=panel,
                               spectrum=spectrum, seed=220507983, image_index=7)
        bin_bytes = path.read_bytes()
        json_text = path.with_suffix(".json").read_text()
    return {"data": data, "bin": np.frombuffer(bin_bytes, dtype=np.uint8), "json": np.array(json_text)}


HIST_SPECS = [(1, (0.0, 1.0)), (3, (0.1, 0.7)), (64, (-2.5, 7.25)), (1000, (1e-3, 3.0))]


def hist_values(precision: str) -> np.ndarray:
    """Seeded values plus every edge case of the binning rule: exact bin edges, lo and hi
    themselves, neighbours one ulp away, +-inf, NaN, subnormals, signed zeros."""
    rng = np.random.default_rng(42)
    v = [rng.uniform(-3.0, 8.0, 20000), rng.lognormal(0.0, 1.0, 5000)]
    for n_bins, (lo, hi) in HIST_SPECS:
        w = (hi - lo) / n_bins
        edges = lo + w * np.arange(n_bins + 1)
        v += [edges, np.nextafter(edges, -np.inf), np.nextafter(edges, np.inf), [lo, hi]]
    v.append([np.inf, -np.inf, np.nan, 5e-324, -5e-324, 0.0, -0.0])
    out = np.concatenate([np.asarray(x, dtype=np.float64) for x in v])
    return out.astype(np.float32) if precision == "f32" else out


def histogram_case():
    """xtrace.kernels.image_histogram (kernels.py:386-430) on hist_values for every spec."""
    res = {}
    for precision in ("f32", "f64"):
        vals = hist_values(precision)
        for n_bins, rng_ in HIST_SPECS:
            h = xk.image_histogram(xk.PixelBuffer((1, vals.size), precision, vals), n_bins, rng_)
            key = f"{precision}_{n_bins}"
            res[key + "_counts"] = h.counts
            res[key + "_cumulative"] = h.cumulative
            res[key + "_under_over"] = np.array([h.underflow, h.overflow])
    return res


def stats_special_values():
    """Non-finite placements for image_stats: NaN in the first / a middle / the last block,
    +-inf, NaN with inf, and signed zeros (block length 8192, 5 blocks)."""
    rng = np.random.default_rng(3)
    base = rng.uniform(-1.0, 1.0, 5 * 8192 - 100)
    cases = []
    for spec in (("nan", 5), ("nan", 20000), ("nan", base.size - 1), ("inf", 9000), ("-inf", 30000),
                 ("nan+inf", (100, 17000)), ("zeros", None)):
        v = base.copy()
        kind, at = spec
        if kind == "nan":
            v[at] = np.nan
        elif kind == "inf":
            v[at] = np.inf
        elif kind == "-inf":
            v[at] = -np.inf
        elif kind == "nan+inf":
            v[at[0]] = np.inf
            v[at[1]] = np.nan
        else:
            v = np.where(np.arange(v.size) % 2 == 0, 0.0, -0.0)
        cases.append(v)
    return cases


def stats_special_case():
    res = {}
    for precision in ("f32", "f64"):
        rows = []
        for v in stats_special_values():
            vv = v.astype(np.float32 if precision == "f32" else np.float64)
            st = xk.image_stats(xk.PixelBuffer((1, vv.size), precision, vv))
            rows.append([st.min, st.max, st.mean, st.total])
        res[precision] = np.array(rows)
    return res


def main(names):
    OUT.mkdir(parents=True, exist_ok=True)
    meta = {}
    for name in names or CASES:
        if name not in CASES:
            continue
        case = CASES[name]
        t0 = time.perf_counter()
        f32, f64 = run_reference(case)
        dt = time.perf_counter() - t0
        arrays = {k: np.asarray(v) for k, v in case.items()}
        np.savez_compressed(OUT / f"{name}.npz", ref_f32=f32, ref_f64=f64, **arrays)
        meta[name] = {"pixels": int(f32.size), "ref_seconds": round(dt, 2), "total_f64": float(f64.sum()),
                      "max_f64": float(f64.max())}
        print(name, meta[name], flush=True)
    for name in names or BG_CASES:
        if name not in BG_CASES:
            continue
        case = BG_CASES[name]
        f32, f64 = run_reference_bg(case)
        np.savez_compressed(OUT / f"{name}.npz", ref_bg_f32=f32, ref_bg_f64=f64,
                            **{k: np.asarray(v) for k, v in case.items()})
        meta[name] = {"pixels": int(f32.size), "total_f64": float(f64.sum())}
        print(name, meta[name], flush=True)
    if not names or "pipeline_full" in names:
        case, acc = pipeline_case()
        np.savez_compressed(OUT / "pipeline_full.npz", ref_image=acc, **{k: np.asarray(v) for k, v in case.items()})
        meta["pipeline_full"] = {"pixels": int(acc.size), "total": float(acc.sum())}
        print("pipeline_full", meta["pipeline_full"], flush=True)
    if not names or "sim_config" in names:
        case = sim_config_case()
        np.savez_compressed(OUT / "sim_config.npz", **case)
        meta["sim_config"] = {"images": len(SIM_SEEDS), "total": float(case["ref_images"].sum())}
        print("sim_config", meta["sim_config"], flush=True)
    if not names or "image_io" in names:
        case = image_io_case()
        np.savez_compressed(OUT / "image_io.npz", **case)
        meta["image_io"] = {"bytes": int(case["bin"].size)}
        print("image_io", meta["image_io"], flush=True)
    if not names or "histogram" in names:
        case = histogram_case()
        np.savez_compressed(OUT / "histogram.npz", **case)
        meta["histogram"] = {"specs": [list(map(str, x)) for x in HIST_SPECS], "generator": "hist_values"}
        print("histogram", len(case), flush=True)
    if not names or "stats_special" in names:
        case = stats_special_case()
        np.savez_compressed(OUT / "stats_special.npz", **case)
        meta["stats_special"] = {"cases": int(case["f64"].shape[0]), "generator": "stats_special_values"}
        print("stats_special", case["f64"].tolist(), flush=True)
    if not names or "stats" in names:
        case = stats_case()
        np.savez_compressed(OUT / "stats.npz", **case)
        meta["stats"] = {"arrays": len(STATS_SPECS), "generator": "tools/make_golden.py:stats_values"}
        print("stats", case["ref_stats"].tolist(), flush=True)
    old = json.loads((OUT / "index.json").read_text()) if (OUT / "index.json").exists() else {}
    old.update(meta)
    (OUT / "index.json").write_text(json.dumps(old, indent=1, sort_keys=True) + "\n")


if __name__ == "__main__":
    main(sys.argv[1:])
