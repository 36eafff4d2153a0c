"""Where the e2e time of one C2 image goes: host descriptor, plan build/upload, kernel, image download."""
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch

from paper_2205_07976_b200 import PixelBuffer, SpotsPlan, describe, nanobragg_spots, synthetic
from paper_2205_07976_b200 import _native as N

compute = sys.argv[1] if len(sys.argv) > 1 else "fp32"
panel = synthetic.rayonix_panel()
ctxs = [synthetic.ls49_context(synthetic.SEED + 1000 + i, panel=panel, compute=compute) for i in range(4)]
img = PixelBuffer.zeros(panel.dims, "f32")
nanobragg_spots(ctxs[0], img)  # warm
for c in ctxs[1:]:
    t0 = time.perf_counter()
    d = describe(c)
    t1 = time.perf_counter()
    plan = SpotsPlan(c)
    torch.cuda.synchronize()
    t2 = time.perf_counter()
    dev = torch.empty(plan.n_pixels, dtype=torch.float32, device="cuda")
    plan.run(dev.data_ptr(), mode=N.OUT_F32, on_device=True)
    t3 = time.perf_counter()
    host = img.data
    t4 = time.perf_counter()
    host[...] = dev.cpu().numpy()  # pageable copy path through torch
    t5 = time.perf_counter()
    pinned = torch.empty(plan.n_pixels, dtype=torch.float32, pin_memory=True)
    t6 = time.perf_counter()
    pinned.copy_(dev)
    torch.cuda.synchronize()
    t7 = time.perf_counter()
    t8 = time.perf_counter()
    nanobragg_spots(c, img)
    t9 = time.perf_counter()
    print(f"describe {1e3*(t1-t0):.2f} ms | plan build+upload {1e3*(t2-t1):.2f} | kernel {plan.kernel_ms:.2f} "
          f"(wall {1e3*(t3-t2):.2f}) | D2H pageable {1e3*(t5-t4):.2f} | D2H pinned {1e3*(t7-t6):.2f} | "
          f"nanobragg_spots wall {1e3*(t9-t8):.2f}", flush=True)
    plan.close()
