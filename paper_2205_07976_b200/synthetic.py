"""Synthetic workloads of BASELINE.json's configs.

No datasets travel with the repo, so every benchmark/parity input is built
here from a seed:

  C1  toy cubic cell, 256x256, 1 source, 1 domain            (c1_context)
  C2  LS49-shape image: ferredoxin-like monoclinic cell, N=30, 3840^2 Rayonix-like
      panel, 100 channels, 50 mosaic domains                  (ls49_context)
  C3  batch of C2 images with per-image orientation/mosaic/weights (ls49_context(seed=SEED+i))
  C4  Jungfrau-16M-like: 256 coplanar 254^2 panels, os=2, 3 thickness layers, FP64
                                                              (jungfrau_context)
  C5  C2 with 1000 channels, sharded by channel               (ls49_context(n_channels=1000, de=0.2, e0=7020))

Values marked "builder-fixed" are synthetic choices, not measured data.
"""
from __future__ import annotations

import math

import numpy as np

from .kernels import SpotsContext
from .model import (
    BeamSpectrum,
    CrystalModel,
    Detector,
    DetectorPanel,
    MosaicDomainSet,
    Orientation,
    StructureFactorTable,
    UnitCell,
    generate_mosaic_rotations,
    reciprocal_basis,
)

SEED = 220507976
HC_EV_A = 12398.419843  # h c in eV * Angstrom

LS49_CELL = (67.2, 59.8, 47.2, 90.0, 113.2, 90.0)  # builder-fixed ferredoxin-like
LS49_NCELLS = (30, 30, 30)


def random_rotation(rng: np.random.Generator) -> np.ndarray:
    """Uniform SO(3) sample from a normalised 4-normal quaternion."""
    q = rng.normal(size=4)
    w, x, y, z = q / np.linalg.norm(q)
    return np.array([
        [1 - 2 * (y * y + z * z), 2 * (x * y - z * w), 2 * (x * z + y * w)],
        [2 * (x * y + z * w), 1 - 2 * (x * x + z * z), 2 * (y * z - x * w)],
        [2 * (x * z - y * w), 2 * (y * z + x * w), 1 - 2 * (x * x + y * y)],
    ])


def wilson_table(cell: UnitCell, dmin: float, seed: int, f000: float = 500.0,
                 default_f: float = 0.0) -> StructureFactorTable:
    """All (h, k, l) with d >= dmin, |F| = 100 sqrt(-ln U) (acentric Wilson), seeded."""
    rs = reciprocal_basis(cell)
    smax = 1.0 / dmin
    # bound each index by |h| <= smax / |row of the inverse-metric projection|
    g = rs @ rs.T
    ginv = np.linalg.inv(g)
    lim = [int(math.floor(smax * math.sqrt(ginv[i, i]))) for i in range(3)]
    hh, kk, ll = np.meshgrid(*(np.arange(-m, m + 1) for m in lim), indexing="ij")
    hkl = np.stack([hh.ravel(), kk.ravel(), ll.ravel()], axis=1)
    s = hkl @ rs
    keep = np.einsum("ij,ij->i", s, s) <= smax * smax
    hkl = hkl[keep]
    rng = np.random.default_rng(seed)
    amp = 100.0 * np.sqrt(-np.log(rng.uniform(1e-12, 1.0, size=len(hkl))))
    entries = {tuple(int(v) for v in t): float(a) for t, a in zip(hkl, amp)}
    entries[(0, 0, 0)] = f000
    return StructureFactorTable(entries, default_f=default_f)


_TABLE_CACHE: dict = {}


def ls49_table(seed: int = SEED) -> StructureFactorTable:
    key = ("ls49", seed)
    if key not in _TABLE_CACHE:
        _TABLE_CACHE[key] = wilson_table(UnitCell(*LS49_CELL), 1.6, seed)
    return _TABLE_CACHE[key]


def ls49_spectrum(n_channels: int = 100, e0: float = 7070.0, de: float = 1.0, seed: int = SEED,
                  fluence: float = 1e24) -> BeamSpectrum:
    """Channels E_j = e0 + j de; weights exp(-0.5((E - 7120)/15)^2)(1 + 0.3 u_j)."""
    rng = np.random.default_rng(seed + 1)
    e = e0 + de * np.arange(n_channels)
    u = rng.uniform(-1.0, 1.0, size=n_channels)
    w = np.exp(-0.5 * ((e - 7120.0) / 15.0) ** 2) * (1.0 + 0.3 * u)
    w = np.maximum(w, 1e-300)
    return BeamSpectrum(samples=tuple(zip((HC_EV_A / e).tolist(), w.tolist())), fluence=fluence,
                        polarization_on=True)


def rayonix_panel(size: int = 3840) -> DetectorPanel:
    """Rayonix-like square panel: 88.6 um pixels at 141.7 mm, beam at the centre."""
    c = (size - 1) / 2.0
    return DetectorPanel(size, size, 88.6e-6, 0.1417, (c, c))


def roi(panel: DetectorPanel, r0: int, c0: int, rows: int, cols: int) -> DetectorPanel:
    """Sub-panel [r0, r0+rows) x [c0, c0+cols) with the same geometry (shifted beam centre).

    Identical pixels to the full panel's (the reference computes every pixel
    independently); used for bounded oracle / CPU-baseline samples.
    """
    return DetectorPanel(rows, cols, panel.pixel_size, panel.distance,
                         (panel.beam_center[0] - r0, panel.beam_center[1] - c0),
                         fast_axis=panel.fast_axis, slow_axis=panel.slow_axis, thickness=panel.thickness,
                         thick_steps=panel.thick_steps, attenuation_length=panel.attenuation_length)


def ls49_crystal(seed: int = SEED, n_domains: int = 50, spread_deg: float = 0.05,
                 table_seed: int = SEED) -> CrystalModel:
    rng = np.random.default_rng(seed)
    return CrystalModel(
        cell=UnitCell(*LS49_CELL),
        orientation=Orientation(random_rotation(rng)),
        n_cells=LS49_NCELLS,
        mosaic=generate_mosaic_rotations(seed, spread_deg, n_domains),
        sf_table=ls49_table(table_seed),
    )


def ls49_context(seed: int = SEED, *, n_channels: int = 100, n_domains: int = 50, e0: float = 7070.0,
                 de: float = 1.0, panel=None, compute: str = "fp32", oversample: int = 1) -> SpotsContext:
    """C2 (and C3/C5 with other seeds / channel counts)."""
    return SpotsContext(
        ls49_crystal(seed, n_domains),
        panel if panel is not None else rayonix_panel(),
        ls49_spectrum(n_channels, e0, de, seed),
        oversample=oversample,
        compute=compute,
    )


def c1_context(compute: str = "fp64") -> SpotsContext:
    """C1: mirrors the reference's acceptance toy (test_acceptance.py:52-65)."""
    crystal = CrystalModel(
        cell=UnitCell(100.0, 100.0, 100.0, 90.0, 90.0, 90.0),
        orientation=Orientation(),
        n_cells=(5, 5, 5),
        mosaic=MosaicDomainSet(np.eye(3)[None, :, :]),
        sf_table=StructureFactorTable({(1, 0, 0): 250.0}, default_f=100.0),
    )
    panel = DetectorPanel(256, 256, 100e-6, 0.1, (127.5, 127.5))
    beam = BeamSpectrum(samples=((1.0, 1.0),), fluence=1e24, polarization_on=True)
    return SpotsContext(crystal, panel, beam, oversample=1, compute=compute)


def jungfrau_detector(n_side: int = 16, size: int = 254, gap: int = 4, pixel: float = 75e-6,
                      distance: float = 0.12, thickness: float = 320e-6, thick_steps: int = 3,
                      attenuation_length: float = 60e-6) -> Detector:
    """C4: n_side^2 coplanar size^2 panels tiled with `gap`-pixel gaps, beam at the tiling centre.

    Si sensor 320 um thick, 3 parallax layers; attenuation length builder-fixed.
    """
    pitch = size + gap
    centre = (n_side * pitch - gap) / 2.0
    panels = []
    for r in range(n_side):
        for c in range(n_side):
            panels.append(DetectorPanel(size, size, pixel, distance, (centre - r * pitch, centre - c * pitch),
                                        thickness=thickness, thick_steps=thick_steps,
                                        attenuation_length=attenuation_length))
    return Detector(tuple(panels))


def jungfrau_context(seed: int = SEED, *, n_side: int = 16, n_channels: int = 100, n_domains: int = 50,
                     compute: str = "fp64") -> SpotsContext:
    return SpotsContext(
        ls49_crystal(seed, n_domains),
        jungfrau_detector(n_side),
        ls49_spectrum(n_channels, 7070.0, 1.0, seed),
        oversample=2,
        compute=compute,
    )
