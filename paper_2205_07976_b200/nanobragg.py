"""nanoBragg-style facade: ``add_nanoBragg_spots()`` and ``raw_pixels``.

``BASELINE.json``'s north star names the CCTBX ``simtbx.nanoBragg`` calls
(``add_nanoBragg_spots``, ``raw_pixels``); the reference package itself only
exposes the xtrace API.  This class maps the nanoBragg-style
setters onto a SpotsContext and runs the same GPU kernel -- no separate
numerics.  Units follow nanoBragg (mm, Angstrom, degrees); ``raw_pixels`` is
a float64 (slow, fast) array that spot calls accumulate into.

    sim = nanoBragg(detpixels_slowfast=(256, 256), pixel_size_mm=0.1, Ncells_abc=(5, 5, 5))
    sim.distance_mm = 100; sim.wavelength_A = 1.0; sim.fluence = 1e24
    sim.unit_cell_tuple = (100, 100, 100, 90, 90, 90)
    sim.Fhkl_tuple = ([(1, 0, 0)], [250.0]); sim.default_F = 100
    sim.add_nanoBragg_spots()
    img = sim.raw_pixels
"""
from __future__ import annotations

import numpy as np

from .kernels import R_E_SQR, PixelBuffer, SpotsContext, add_noise, nanobragg_spots
from .model import (
    BeamSpectrum,
    CrystalModel,
    DetectorPanel,
    MosaicDomainSet,
    Orientation,
    PhiScan,
    StructureFactorTable,
    UnitCell,
    generate_mosaic_rotations,
)

__all__ = ["nanoBragg", "shapetype"]


class shapetype:
    """Crystal shape-transform selector (nanoBragg's shapetype enum)."""

    Square = "sincg"
    Gauss = "gauss"
    Round = "round"
    Tophat = "tophat"


class nanoBragg:
    def __init__(self, detpixels_slowfast=(1024, 1024), pixel_size_mm=0.1, Ncells_abc=(1, 1, 1), verbose=0,
                 oversample=1):
        self.detpixels_slowfast = (int(detpixels_slowfast[0]), int(detpixels_slowfast[1]))
        self.pixel_size_mm = float(pixel_size_mm)
        self.Ncells_abc = tuple(int(x) for x in Ncells_abc)
        self.verbose = verbose
        self.oversample = int(oversample)
        self.distance_mm = 100.0
        s, f = self.detpixels_slowfast
        # direct beam on the panel centre (pixel-centre convention of the reference)
        self.beam_center_mm = (s / 2.0 * self.pixel_size_mm, f / 2.0 * self.pixel_size_mm)
        self.fast_axis = (1.0, 0.0, 0.0)
        self.slow_axis = (0.0, 1.0, 0.0)
        self.beam_vector = (0.0, 0.0, 1.0)
        self.wavelength_A = 1.0
        self.spectrum = None              # list of (wavelength_A, weight); overrides wavelength_A
        self.fluence = 1e24               # photons / m^2
        self.polarization_on = True
        self.unit_cell_tuple = (100.0, 100.0, 100.0, 90.0, 90.0, 90.0)
        self.Umatrix = np.eye(3)
        self.mosaic_spread_deg = 0.0
        self.mosaic_domains = 1
        self.mosaic_seed = 0
        self.mosaic_rotations = None      # explicit (n, 3, 3) list wins over the seeded draw
        self.Fhkl_tuple = ((), ())
        self.default_F = 0.0
        self.xtal_shape = shapetype.Square
        self.detector_thick_mm = 0.0
        self.detector_thicksteps = 1
        self.detector_attenuation_length_mm = 0.0
        self.phi_deg = 0.0
        self.osc_deg = 0.0
        self.phisteps = 1
        self.spindle_axis = (1.0, 0.0, 0.0)
        self.seed = 0
        self.compute = "fp64"
        self.raw_pixels = np.zeros(self.detpixels_slowfast, dtype=np.float64)

    # -- derived convenience ----------------------------------------------------
    def set_flux(self, flux_photons_per_s: float, exposure_s: float, beamsize_mm: float):
        """fluence = flux * exposure / beamsize^2 (nanoBragg's definition)."""
        self.fluence = flux_photons_per_s * exposure_s / (beamsize_mm * 1e-3) ** 2

    def panel(self) -> DetectorPanel:
        ps_m = self.pixel_size_mm * 1e-3
        s, f = self.detpixels_slowfast
        bc = (self.beam_center_mm[0] / self.pixel_size_mm, self.beam_center_mm[1] / self.pixel_size_mm)
        return DetectorPanel(
            s, f, ps_m, self.distance_mm * 1e-3, bc, fast_axis=tuple(self.fast_axis),
            slow_axis=tuple(self.slow_axis), thickness=self.detector_thick_mm * 1e-3,
            thick_steps=self.detector_thicksteps, attenuation_length=self.detector_attenuation_length_mm * 1e-3,
        )

    def crystal(self) -> CrystalModel:
        if self.mosaic_rotations is not None:
            mosaic = MosaicDomainSet(np.asarray(self.mosaic_rotations, dtype=float))
        else:
            mosaic = generate_mosaic_rotations(self.mosaic_seed, self.mosaic_spread_deg, self.mosaic_domains)
        indices, amps = self.Fhkl_tuple
        return CrystalModel(
            cell=UnitCell(*self.unit_cell_tuple),
            orientation=Orientation(self.Umatrix),
            n_cells=self.Ncells_abc,
            mosaic=mosaic,
            sf_table=StructureFactorTable(dict(zip((tuple(i) for i in indices), amps)), default_f=self.default_F),
        )

    def beam(self) -> BeamSpectrum:
        samples = self.spectrum if self.spectrum is not None else [(self.wavelength_A, 1.0)]
        return BeamSpectrum(samples=tuple(samples), fluence=self.fluence, polarization_on=self.polarization_on,
                            beam_direction=tuple(self.beam_vector))

    def to_context(self) -> SpotsContext:
        phi = None
        if self.phisteps != 1 or self.phi_deg != 0.0 or self.osc_deg != 0.0:
            phi = PhiScan(self.phi_deg, self.osc_deg, self.phisteps, tuple(self.spindle_axis))
        return SpotsContext(self.crystal(), self.panel(), self.beam(), oversample=self.oversample,
                            r_e_sqr=R_E_SQR, compute=self.compute, shape=self.xtal_shape, phi=phi)

    # -- nanoBragg verbs --------------------------------------------------------
    def add_nanoBragg_spots(self):
        """raw_pixels += the Bragg-spot image (computed on the GPU in FP64 store)."""
        buf = PixelBuffer(self.detpixels_slowfast, "f64")
        nanobragg_spots(self.to_context(), buf)
        self.raw_pixels = self.raw_pixels + buf.as_image()

    def add_noise(self, image: int = 0):
        """raw_pixels <- Poisson(raw_pixels), Philox keyed by (seed, image)."""
        buf = PixelBuffer(self.detpixels_slowfast, "f64", self.raw_pixels.reshape(-1))
        self.raw_pixels = add_noise(buf, self.seed, image).as_image().copy()

    def free_all(self):
        self.raw_pixels = np.zeros(self.detpixels_slowfast, dtype=np.float64)
