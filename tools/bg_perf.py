"""Device time of the background stage on the C2 detector (add_background, kernels.py:279-312).

Times nbx_background alone and simulate_image (spots + background fused) vs spots alone.
"""
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch

from paper_2205_07976_b200 import BackgroundProfile, PixelBuffer, SpotsPlan, simulate_image, synthetic
from paper_2205_07976_b200 import _native as N
from paper_2205_07976_b200.kernels import _bg_descriptor

WATER = BackgroundProfile(points=((0.0, 2.57), (0.0365, 2.58), (0.07, 2.8), (0.12, 5.0), (0.162, 8.0), (0.2, 7.5),
                                  (0.25, 7.0), (0.3, 6.5), (0.35, 6.1), (0.4, 5.8), (0.45, 5.5), (0.5, 5.2)))
panel = synthetic.rayonix_panel()
ctx = synthetic.ls49_context(panel=panel, compute="fp32")
cx = N.context()
dev = torch.zeros(panel.n_pixels, dtype=torch.float32, device="cuda")
desc = _bg_descriptor(WATER, panel, ctx.spectrum, 1.0)
bad = N.C.c_int64(-1)
for _ in range(2):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    st = cx.lib.nbx_background(cx.handle, N.C.byref(desc.c), N.OUT_F32, dev.data_ptr(), 1, N.C.byref(bad))
    torch.cuda.synchronize()
    print(f"nbx_background C2 ({len(WATER.points)}-point profile, 100 channels): {1e3 * (time.perf_counter() - t0):.2f} ms "
          f"wall (status {st})", flush=True)
plan = SpotsPlan(ctx)
img = torch.zeros(panel.n_pixels, dtype=torch.float64, device="cuda")
for mode, name in ((N.OUT_F32, "spots only"), (N.OUT_IMAGE_F64, "spots+background fused (no profile in plan)")):
    plan.run(img.data_ptr() if mode != N.OUT_F32 else dev.data_ptr(), mode=mode, on_device=True)
    print(f"{name}: {plan.kernel_ms:.2f} ms", flush=True)
out = PixelBuffer.zeros(panel.dims, "f64")
for _ in range(2):
    t0 = time.perf_counter()
    simulate_image(ctx, background=WATER, out=out)
    print(f"simulate_image (host buffers, spots+background fused): {1e3 * (time.perf_counter() - t0):.2f} ms", flush=True)
