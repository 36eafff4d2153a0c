"""Shared parity helpers for the tests (test infrastructure).

golden(name) rebuilds the package's inputs from a fixture written by
tools/make_golden.py (which ran the reference itself); the metrics follow
SURVEY.md §8 D1: relative error of the TOTAL and of every SPOT (8-connected
components of oracle >= 1e-3 max), plus per-pixel diagnostics.
"""
from __future__ import annotations

from pathlib import Path

import numpy as np

from paper_2205_07976_b200 import (
    BeamSpectrum,
    CrystalModel,
    DetectorPanel,
    MosaicDomainSet,
    Orientation,
    SpotsContext,
    StructureFactorTable,
    UnitCell,
)

GOLDEN = Path(__file__).resolve().parent / "golden"


def load(name: str) -> dict:
    z = np.load(GOLDEN / f"{name}.npz")
    return {k: z[k] for k in z.files}


def context(case: dict, compute: str = "fp64", **kw) -> SpotsContext:
    crystal = CrystalModel(
        cell=UnitCell(*[float(x) for x in case["cell"]]),
        orientation=Orientation(case["orientation"]),
        n_cells=tuple(int(x) for x in case["n_cells"]),
        mosaic=MosaicDomainSet(case["mosaic"]),
        sf_table=StructureFactorTable(
            {tuple(int(v) for v in h): float(a) for h, a in zip(case["hkl"], case["amp"])},
            default_f=float(case["default_f"])),
    )
    p = case["panel"]
    panel = DetectorPanel(int(p[0]), int(p[1]), float(p[2]), float(p[3]), (float(p[4]), float(p[5])),
                          fast_axis=tuple(float(x) for x in case["fast_axis"]),
                          slow_axis=tuple(float(x) for x in case["slow_axis"]))
    beam = BeamSpectrum(samples=tuple(map(tuple, case["samples"].tolist())), fluence=float(case["fluence"]),
                        polarization_on=bool(case["pol"]),
                        beam_direction=tuple(float(x) for x in case["beam_dir"]))
    return SpotsContext(crystal, panel, beam, oversample=int(case["oversample"]), compute=compute, **kw)


def spot_labels(ref: np.ndarray, dims, frac: float = 1e-3):
    from scipy import ndimage

    img = ref.reshape(dims)
    mask = img >= frac * img.max()
    labels, n = ndimage.label(mask, structure=np.ones((3, 3)))
    return labels, n


def metrics(got: np.ndarray, ref: np.ndarray, dims) -> dict:
    got = np.asarray(got, dtype=np.float64).reshape(-1)
    ref = np.asarray(ref, dtype=np.float64).reshape(-1)
    tot = abs(got.sum() - ref.sum()) / abs(ref.sum()) if ref.sum() != 0 else abs(got.sum())
    if ref.max() <= 0:
        z = float(np.abs(got).max())
        return {"total": tot, "spot": z, "n_spots": 0, "pix_abs_over_max": z, "pix_rel_bright": z}
    labels, n = spot_labels(ref, dims)
    spot = 0.0
    if n:
        from scipy import ndimage

        idx = np.arange(1, n + 1)
        rs = ndimage.sum(ref.reshape(dims), labels, idx)
        gs = ndimage.sum(got.reshape(dims), labels, idx)
        spot = float(np.max(np.abs(gs - rs) / np.abs(rs)))
    mx = ref.max() if ref.max() > 0 else 1.0
    bright = ref >= 1e-3 * mx
    pix_rel = float(np.max(np.abs(got[bright] - ref[bright]) / ref[bright])) if bright.any() else 0.0
    return {"total": float(tot), "spot": spot, "n_spots": int(n),
            "pix_abs_over_max": float(np.max(np.abs(got - ref)) / mx), "pix_rel_bright": pix_rel}


def bg_inputs(case: dict):
    """(profile, panel, spectrum, thickness_factor) of a background fixture."""
    from paper_2205_07976_b200 import BackgroundProfile

    p = case["panel"]
    panel = DetectorPanel(int(p[0]), int(p[1]), float(p[2]), float(p[3]), (float(p[4]), float(p[5])),
                          fast_axis=tuple(float(x) for x in case["fast_axis"]),
                          slow_axis=tuple(float(x) for x in case["slow_axis"]))
    beam = BeamSpectrum(samples=tuple(map(tuple, case["samples"].tolist())), fluence=float(case["fluence"]),
                        polarization_on=bool(case["pol"]),
                        beam_direction=tuple(float(x) for x in case["beam_dir"]))
    prof = BackgroundProfile(points=tuple(map(tuple, case["bg_points"].tolist())))
    return prof, panel, beam, float(case["thickness_factor"])
