"""Host-side latency of the drop-in call on small images (C1 toy, a 256^2 LS49 ROI) and of describe()."""
import sys, time
sys.path.insert(0, '.')
import numpy as np
from paper_2205_07976_b200 import PixelBuffer, nanobragg_spots, synthetic, describe
ctx = synthetic.c1_context()
out = PixelBuffer.zeros(ctx.panel.dims, "f32")
for i in range(3): nanobragg_spots(ctx, out)
t=[]
for i in range(50):
    t0=time.perf_counter(); nanobragg_spots(ctx, out); t.append(time.perf_counter()-t0)
print("C1 nanobragg_spots median ms", 1e3*np.median(t))
t=[]
for i in range(50):
    t0=time.perf_counter(); describe(ctx); t.append(time.perf_counter()-t0)
print("describe median ms", 1e3*np.median(t))
ctx2 = synthetic.ls49_context(panel=synthetic.roi(synthetic.rayonix_panel(), 1800, 1800, 256, 256))
out2 = PixelBuffer.zeros(ctx2.panel.dims, "f32")
for i in range(3): nanobragg_spots(ctx2, out2)
t=[]
for i in range(20):
    t0=time.perf_counter(); nanobragg_spots(ctx2, out2); t.append(time.perf_counter()-t0)
print("LS49 256^2 ROI median ms", 1e3*np.median(t))
t=[]
for i in range(20):
    t0=time.perf_counter(); describe(ctx2); t.append(time.perf_counter()-t0)
print("describe ls49 median ms", 1e3*np.median(t))
