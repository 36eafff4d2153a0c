"""Host-side latency of the drop-in call on small images (C1 toy, a 256^2 LS49 ROI) and of describe().

usage: python tools/call_latency.py
"""
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np

from paper_2205_07976_b200 import PixelBuffer, describe, nanobragg_spots, synthetic


def median_ms(fn, n):
    t = []
    for _ in range(n):
        t0 = time.perf_counter()
        fn()
        t.append(time.perf_counter() - t0)
    return 1e3 * float(np.median(t))


cases = {
    "C1 toy 256^2": synthetic.c1_context(),
    "LS49 256^2 ROI": synthetic.ls49_context(panel=synthetic.roi(synthetic.rayonix_panel(), 1800, 1800, 256, 256)),
}
for name, ctx in cases.items():
    out = PixelBuffer.zeros(ctx.panel.dims, "f32")
    for _ in range(3):
        nanobragg_spots(ctx, out)
    print(f"{name}: nanobragg_spots {median_ms(lambda: nanobragg_spots(ctx, out), 30):.3f} ms, "
          f"describe {median_ms(lambda: describe(ctx), 30):.3f} ms", flush=True)
