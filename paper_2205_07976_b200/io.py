"""Image pipeline around the spot kernel: campaign rendering and the .bin/.json format.

SURVEY §8 F3 (the caller of the hot path) and F4 (image statistics):

* ``write_image`` / ``read_image`` restate the reference's on-disk format
  (/root/reference/pkg/src/xtrace/io.py:403-456): ``<stem>.bin`` raw
  little-endian float32, ``<stem>.json`` sidecar with dims, dtype, geometry,
  seed, image index and the zlib CRC-32 of the payload.
* ``run_campaign`` renders many images through ``nbx_campaign``: each image is
  simulate_image's accumulator (spots + optional background) rounded to the
  float32 payload ON the device, and the kernel of image i+1 runs while image
  i is copied, checksummed (native CRC-32) and written -- the reference's
  device-slot / I/O overlap (scheduler.py:190-247) done with streams.  Under
  torch.distributed each rank renders its contiguous block of indices
  (plan_batches, scheduler.py:138-153).  File names: ``img_{index:06d}``.
* ``image_stats`` / ``image_histogram``: device reduce / histogram with the
  reference's result types (kernels.py:334-430).
"""
from __future__ import annotations

import ctypes as C
import json
import zlib
from dataclasses import dataclass
from pathlib import Path
from typing import Callable, NamedTuple

import numpy as np

from . import _native as N
from .errors import CampaignIOError, NumericalFault, ShapeMismatchError
from .kernels import PixelBuffer, describe

__all__ = ["write_image", "read_image", "run_campaign", "campaign_indices", "CampaignResult", "image_stats", "image_histogram",
           "ImageStats", "HistogramResult", "image_stem"]

_DOWNCAST = "values rounded to nearest-even from the float64 accumulator"


def _stem(path) -> Path:
    path = Path(path)
    return path.with_suffix("") if path.suffix in (".bin", ".json") else path


def image_stem(out_dir, index: int) -> Path:
    return Path(out_dir) / f"img_{index:06d}"


def _sidecar(dims, crc, panel=None, spectrum=None, seed=None, image_index=None) -> dict:
    return {
        "dims": list(dims),
        "dtype": "float32",
        "byte_order": "little",
        "downcast": _DOWNCAST,
        "pixel_size_m": panel.pixel_size if panel is not None and hasattr(panel, "pixel_size") else None,
        "distance_m": panel.distance if panel is not None and hasattr(panel, "distance") else None,
        "wavelengths_angstrom": list(map(float, spectrum.wavelengths)) if spectrum is not None else None,
        "seed": seed,
        "image_index": image_index,
        "crc32": int(crc),
    }


def _write_sidecar(stem: Path, sidecar: dict):
    with open(stem.with_suffix(".json"), "w", encoding="utf-8") as fh:
        json.dump(sidecar, fh, indent=1)
        fh.write("\n")


def write_image(buf: PixelBuffer, path, panel=None, spectrum=None, seed: int | None = None,
                image_index: int | None = None) -> Path:
    """``<stem>.bin`` (little-endian float32) + ``<stem>.json`` (io.py:403-434); refuses non-finite data."""
    finite = np.isfinite(buf.data)
    if not finite.all():
        raise NumericalFault(int(np.argmin(finite)), "refusing to write non-finite pixel")
    stem = _stem(path)
    payload = np.ascontiguousarray(buf.data, dtype="<f4").tobytes()
    bin_path = stem.with_suffix(".bin")
    with open(bin_path, "wb") as fh:
        fh.write(payload)
    _write_sidecar(stem, _sidecar(buf.dims, zlib.crc32(payload), panel, spectrum, seed, image_index))
    return bin_path


def read_image(path, verify_crc: bool = True) -> tuple[np.ndarray, dict]:
    """Read a .bin image and its sidecar back, checking the CRC (io.py:437-456)."""
    stem = _stem(path)
    sidecar_path = stem.with_suffix(".json")
    if not sidecar_path.exists():
        raise FileNotFoundError(f"missing sidecar {sidecar_path}")
    sidecar = json.loads(sidecar_path.read_text(encoding="utf-8"))
    payload = stem.with_suffix(".bin").read_bytes()
    if verify_crc and zlib.crc32(payload) != sidecar["crc32"]:
        raise ValueError(f"CRC mismatch for {stem.with_suffix('.bin')}")
    dims = tuple(sidecar["dims"])
    data = np.frombuffer(payload, dtype="<f4")
    if data.size != dims[0] * dims[1]:
        raise ValueError(f"payload length {data.size} != dims {dims}")
    return data.reshape(dims), sidecar


@dataclass
class CampaignResult:
    """Images written (index, .bin path, payload CRC-32, in index order) and images flagged.

    ``flagged`` holds (index, lowest non-finite pixel) for every image whose spots or
    background faulted: like the reference's rank loop (scheduler.py:208-214) the image is
    skipped and the campaign carries on.
    """
    indices: list[int]
    paths: list[Path]
    crcs: list[int]
    seconds: float
    flagged: list[tuple[int, int]] = None

    def __post_init__(self):
        if self.flagged is None:
            self.flagged = []


def campaign_indices(n_images: int, first_image: int = 0, group=None) -> list[int]:
    """This rank's images of [first_image, first_image + n_images): its contiguous block of the
    reference's static partition (plan_batches, scheduler.py:138-153) over the ranks of
    ``group`` when torch.distributed is initialised, else all of them."""
    world, rank = 1, 0
    try:
        import torch.distributed as dist

        if dist.is_initialized():
            world, rank = dist.get_world_size(group), dist.get_rank(group)
    except ImportError:
        pass
    from .parallel import plan_batches

    _, (lo, hi) = plan_batches(n_images, world)[rank]
    return list(range(first_image + lo, first_image + hi))


def run_campaign(context_for: Callable[[int], object], n_images: int, out_dir, *, first_image: int = 0,
                 background=None, thickness_factor: float = 1.0, seeds: Callable[[int], int] | None = None,
                 group=None, device: int | None = None) -> CampaignResult:
    """Render images [first_image, first_image + n_images) (this rank's share) and write them.

    ``context_for(index)`` returns the SpotsContext of image ``index`` (e.g. a
    per-image seed, like SimulationConfig.crystal_for_seed, io.py:146-157).  Like the
    reference's rank loop (scheduler.py:190-247): an image whose spots or background are
    non-finite is flagged in ``CampaignResult.flagged`` and skipped, the others are written;
    a file that cannot be written raises CampaignIOError after the sidecars of every image
    written before it; a non-finite float32 payload raises NumericalFault (write_image).
    """
    import time

    indices = campaign_indices(n_images, first_image, group)
    out_dir = Path(out_dir)
    out_dir.mkdir(parents=True, exist_ok=True)
    ctxs = [context_for(i) for i in indices]
    descs = [describe(c, background=background, thickness_factor=thickness_factor) for c in ctxs]
    stems = [image_stem(out_dir, i) for i in indices]
    paths = [s.with_suffix(".bin") for s in stems]
    cx = N.context(device)
    n = len(indices)
    arr = (N.SpotsDesc * max(n, 1))(*[d.c for d in descs])
    cpaths = (C.c_char_p * max(n, 1))(*[str(p).encode() for p in paths])
    crcs = (C.c_uint32 * max(n, 1))()
    faults = (C.c_int64 * max(n, 1))()
    compute = N.COMPUTE[getattr(ctxs[0], "compute", "fp64")] if ctxs else 0
    t0 = time.perf_counter()
    with cx.lock:
        status = cx.lib.nbx_campaign(cx.handle, arr, n, compute, cpaths, crcs, faults)
        msg = cx.error() if status != N.NBX_OK else ""
    seconds = time.perf_counter() - t0
    if status not in (N.NBX_OK, N.NBX_ERR_NUMERICAL, N.NBX_ERR_IO):
        if status == N.NBX_ERR_ARG:
            raise ShapeMismatchError(msg) if "dims" in msg or "buffer" in msg else ValueError(msg)
        raise N.NativeError(msg)
    done, flagged = [], []
    for i in range(n):
        f = int(faults[i])
        if f == -1:  # written: its sidecar (write_image writes .bin then .json, io.py:425-433)
            _write_sidecar(stems[i], _sidecar(ctxs[i].panel.dims, crcs[i], ctxs[i].panel, ctxs[i].spectrum,
                                              seeds(indices[i]) if seeds else None, indices[i]))
            done.append(i)
        elif f >= 0 and (f >> 40) in (0, 1):
            flagged.append((indices[i], f & ((1 << 40) - 1)))
    if status == N.NBX_ERR_NUMERICAL:  # a non-finite float32 payload: write_image refuses it (io.py:409-411)
        i = next(j for j in range(n) if int(faults[j]) >= 0 and (int(faults[j]) >> 40) == 2)
        pix = int(faults[i]) & ((1 << 40) - 1)
        raise NumericalFault(pix, f"image {indices[i]}: refusing to write non-finite pixel {pix}")
    if status == N.NBX_ERR_IO:  # the reference aborts the campaign (scheduler.py:219-225)
        i = next(j for j in range(n) if int(faults[j]) == -3)
        raise CampaignIOError(indices[i], msg)
    return CampaignResult([indices[i] for i in done], [paths[i] for i in done], [int(crcs[i]) for i in done],
                          seconds, flagged)


class ImageStats(NamedTuple):
    min: float
    max: float
    mean: float
    total: float


@dataclass(frozen=True)
class HistogramResult:
    counts: np.ndarray
    cumulative: np.ndarray
    underflow: int
    overflow: int

    @property
    def n_binned(self) -> int:
        return int(self.counts.sum())


def _dtype_code(buf: PixelBuffer) -> int:
    return 1 if buf.data.dtype == np.float64 else 0


def image_stats(buf: PixelBuffer, executor=None) -> ImageStats:
    """Exact min/max, fixed-tree mean/total on the device (kernels.py:346-371)."""
    if buf.n_pixels == 0:
        raise ValueError("image_stats requires a non-empty buffer")
    cx = N.context()
    out = (C.c_double * 4)()
    data = np.ascontiguousarray(buf.data)
    with cx.lock:
        status = cx.lib.nbx_image_stats(cx.handle, data.ctypes.data, data.size, _dtype_code(buf), 0, out)
        N.check(cx, status, label="image_stats")
    return ImageStats(out[0], out[1], out[2], out[3])


def image_histogram(buf: PixelBuffer, n_bins: int, value_range: tuple[float, float],
                    executor=None) -> HistogramResult:
    """Counts per bin, top bin closed, under/overflow, inclusive cumulative (kernels.py:386-430)."""
    lo, hi = float(value_range[0]), float(value_range[1])
    if not lo < hi:
        raise ValueError("histogram range must satisfy lo < hi")
    if n_bins < 1:
        raise ValueError("n_bins must be >= 1")
    if buf.n_pixels == 0:
        raise ValueError("image_histogram requires a non-empty buffer")
    cx = N.context()
    counts = np.zeros(n_bins, dtype=np.int64)
    under, over = C.c_int64(0), C.c_int64(0)
    data = np.ascontiguousarray(buf.data)
    with cx.lock:
        status = cx.lib.nbx_image_histogram(cx.handle, data.ctypes.data, data.size, _dtype_code(buf), 0, n_bins,
                                            lo, hi, counts.ctypes.data_as(C.POINTER(C.c_int64)), C.byref(under),
                                            C.byref(over))
        N.check(cx, status, label="image_histogram")
    return HistogramResult(counts, np.cumsum(counts), int(under.value), int(over.value))
