"""Small runs of every kernel variant, for compute-sanitizer (memcheck / racecheck / initcheck).

usage: compute-sanitizer --tool memcheck python tools/sanitize_run.py
Covers: FP32 MUFU / polynomial / degree-4 numerators, FP64 direct, bracket and segmented
recurrences (incl. the direct beam's all-slow channels and span-cut runs), the
non-grating shapes, the wide (integer) index, thickness layers + multi-panel, background
fused into the image, the banded (pipelined) host download, add_array, noise, stats, the
standalone background, the sparse Fhkl table, several FP64 recurrence runs, channel-shard
partials with finalize and the slot reduction, and the pipelined campaign (incl. a flagged image).
"""
import dataclasses
import os
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np

from paper_2205_07976_b200 import (BackgroundProfile, PixelBuffer, SpotsPlan, add_array, add_noise,
                                   nanobragg_spots, simulate_image, synthetic)
from paper_2205_07976_b200 import _native as N
from paper_2205_07976_b200.io import image_histogram, image_stats

WATER = BackgroundProfile(points=((0.0, 2.57), (0.07, 2.8), (0.12, 5.0), (0.3, 6.5)))


def run(ctx, precision="f32"):
    out = PixelBuffer.zeros(ctx.panel.dims, precision)
    nanobragg_spots(ctx, out)
    assert np.all(np.isfinite(out.data))
    return out


roi = synthetic.roi(synthetic.rayonix_panel(), 1890, 1890, 40, 36)
for compute in ("fp32", "fp64"):
    for nch, ndom in ((3, 2), (64, 4)):  # few samples (polynomial / direct) and many (MUFU / recurrence)
        ctx = synthetic.ls49_context(panel=roi, n_channels=nch, n_domains=ndom, compute=compute)
        run(ctx)
        print(compute, nch, ndom, "variant", SpotsPlan(ctx).info.kernel_variant, flush=True)
os.environ["NBX_FP32_POLY"] = "4"
run(synthetic.ls49_context(panel=roi, n_channels=8, n_domains=2, compute="fp32"))
del os.environ["NBX_FP32_POLY"]
os.environ["NBX_FP32_NUM"] = "poly"  # the degree-3 polynomial loop (variant 5)
run(synthetic.ls49_context(panel=roi, n_channels=8, n_domains=2, compute="fp32"))
del os.environ["NBX_FP32_NUM"]
for shape in ("gauss", "round", "tophat"):
    for compute in ("fp32", "fp64"):
        run(dataclasses.replace(synthetic.ls49_context(panel=roi, n_channels=4, n_domains=2, compute=compute),
                                shape=shape))
# multi-panel detector with thickness layers and oversampling
det = synthetic.jungfrau_detector(n_side=2, size=20, thickness=320e-6)
for compute in ("fp32", "fp64"):
    run(dataclasses.replace(synthetic.ls49_context(panel=det, n_channels=4, n_domains=2, compute=compute),
                            oversample=2))
# banded host download (>= 2^20 pixels), ragged last band
big = synthetic.roi(synthetic.rayonix_panel(), 1400, 1400, 1030, 1024)
run(synthetic.ls49_context(panel=big, n_channels=1, n_domains=1, compute="fp32"))
# spots + background fused, add_array, noise, stats
ctx = synthetic.ls49_context(panel=roi, n_channels=4, n_domains=2, compute="fp32")
img = simulate_image(ctx, background=WATER)
spots = run(ctx)
acc = PixelBuffer.zeros(roi.dims, "f64")
add_array(acc, spots)
add_noise(spots, seed=5)
image_stats(img)
image_histogram(img, 16, (0.0, float(img.data.max()) + 1.0))
# standalone background, sparse Fhkl table, FP64 recurrence with several runs
from paper_2205_07976_b200 import add_background  # noqa: E402

bg = PixelBuffer.zeros(roi.dims, "f32")
add_background(WATER, ctx.panel, ctx.spectrum, 1.0, bg)
os.environ["NBX_FHKL_HASH"] = "1"
for compute in ("fp32", "fp64"):
    run(synthetic.ls49_context(panel=roi, n_channels=16, n_domains=2, compute=compute))
del os.environ["NBX_FHKL_HASH"]
two_runs = synthetic.ls49_context(panel=roi, n_channels=200, n_domains=1, compute="fp64")
run(two_runs)
# FP64 kernel variants: the per-channel bracket recurrence and the segmented one on the direct
# beam (S = 0: every channel slow, the limit branch), on a span-cut wide band (several runs)
os.environ["NBX_FP64_REC"] = "1"
run(synthetic.ls49_context(panel=roi, n_channels=64, n_domains=2, compute="fp64"))
del os.environ["NBX_FP64_REC"]
beam_px = synthetic.roi(synthetic.rayonix_panel(), 1915, 1915, 10, 10)
run(synthetic.ls49_context(panel=beam_px, n_channels=32, n_domains=2, compute="fp64"), "f64")
wide = synthetic.roi(synthetic.rayonix_panel(), 0, 0, 8, 40)
run(synthetic.ls49_context(panel=wide, n_channels=100, de=2.0, n_domains=2, compute="fp64"))
# channel shards: RAW partials + finalize, and the peer-memory slot reduction (one process)
import torch  # noqa: E402

whole = SpotsPlan(ctx)
raw = torch.zeros(2 * whole.n_pixels, dtype=torch.float64, device="cuda")
n_src = len(ctx.spectrum.samples)
for r, (lo, hi) in enumerate(((0, n_src // 2), (n_src // 2, n_src))):
    part = SpotsPlan(ctx, src_begin=lo, src_end=hi, norm=0.0)
    part.run(raw.data_ptr() + r * whole.n_pixels * 8, mode=N.OUT_RAW_STORE_F64, on_device=True)
cx = N.context()
out = np.zeros(whole.n_pixels, np.float32)
bad = N.C.c_int64(-1)
assert cx.lib.nbx_reduce_slots(cx.handle, raw.data_ptr(), 2, whole.n_pixels, whole.scale, N.OUT_F32,
                               out.ctypes.data, 0, N.C.byref(bad)) == 0
assert cx.lib.nbx_finalize(cx.handle, raw.data_ptr(), whole.n_pixels, whole.scale, N.OUT_F32, out.ctypes.data, 0,
                           N.C.byref(bad)) == 0
# the pipelined campaign (double-buffered download, CRC-32, file writes)
import tempfile  # noqa: E402

from paper_2205_07976_b200.io import run_campaign  # noqa: E402

with tempfile.TemporaryDirectory() as d:
    run_campaign(lambda i: synthetic.ls49_context(synthetic.SEED + i, panel=roi, n_channels=4, n_domains=2), 3, d,
                 background=WATER)


def hot(i):  # image 1 overflows float32: flagged, the campaign continues
    c = synthetic.ls49_context(synthetic.SEED + i, panel=roi, n_channels=4, n_domains=2)
    return dataclasses.replace(c, spectrum=dataclasses.replace(c.spectrum, fluence=1e64)) if i == 1 else c


with tempfile.TemporaryDirectory() as d:
    assert [f[0] for f in run_campaign(hot, 3, d).flagged] == [1]
print("sanitize run complete", flush=True)
