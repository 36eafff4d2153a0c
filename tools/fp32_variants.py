"""FP32 path: the segmented-index MUFU loop (variant 7, opt-in NBX_FP32_SEG=1 on uniform spectra)
against the per-channel-index MUFU loop (variant 1, the default) on the full C2 image: kernel
times and the largest per-pixel / total / per-spot difference (they differ only in where F^2
multiplies).

usage: python tools/fp32_variants.py [size]
"""
import os
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
sys.path.insert(0, str(Path(__file__).resolve().parents[1] / "tests"))
import numpy as np
import torch

import parity
from paper_2205_07976_b200 import SpotsPlan, synthetic
from paper_2205_07976_b200 import _native as N

args = [a for a in sys.argv[1:] if not a.startswith("--")]
size = int(args[0]) if args else 3840
r0 = (3840 - size) // 2
panel = synthetic.rayonix_panel() if size == 3840 else synthetic.roi(synthetic.rayonix_panel(), r0, r0, size, size)
ctx = synthetic.ls49_context(panel=panel, compute="fp32")
imgs = {}
variants = (("segmented", "1"), ("per-channel", None)) if "--seg-only" not in sys.argv else (("segmented", "1"),)
for name, env in variants:
    if env is None:
        os.environ.pop("NBX_FP32_SEG", None)
    else:
        os.environ["NBX_FP32_SEG"] = env
    p = SpotsPlan(ctx)
    out = torch.empty(p.n_pixels, dtype=torch.float64, device="cuda")
    ms = []
    for _ in range(3):
        p.run(out.data_ptr(), mode=N.OUT_F64, on_device=True)
        ms.append(p.kernel_ms)
    imgs[name] = out.cpu().numpy()
    print(f"C2 {size}^2 FP32 {name} (variant {p.info.kernel_variant}): {[round(m, 2) for m in ms]} ms, "
          f"{p.steps / min(ms) / 1e6:.1f} Gsteps/s", flush=True)
    p.close()
if len(imgs) < 2:
    sys.exit(0)
m = parity.metrics(imgs["segmented"], imgs["per-channel"], panel.dims)
print(f"segmented vs per-channel: total {m['total']:.2e} spot {m['spot']:.2e} pixabs/max {m['pix_abs_over_max']:.2e} "
      f"pixrel(bright) {m['pix_rel_bright']:.2e}", flush=True)
