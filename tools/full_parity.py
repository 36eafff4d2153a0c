"""Full-size (C2, 3840^2 x 100 ch x 50 domains) FP32-path parity against the FP64 path on the GPU.

The FP64 path is pinned to the reference at 1e-9 on the golden ROIs; this
checks the FP32 path's total and per-spot error on the whole benchmark image.
Writes one JSON line (to stdout) per FP32 variant.
"""
import json
import os
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
sys.path.insert(0, str(Path(__file__).resolve().parents[1] / "tests"))
import numpy as np

import parity
from paper_2205_07976_b200 import SpotsPlan, synthetic
from paper_2205_07976_b200 import _native as N

size = int(sys.argv[1]) if len(sys.argv) > 1 else 3840
seed = synthetic.SEED + (int(sys.argv[2]) if len(sys.argv) > 2 else 0)
r0 = (3840 - size) // 2
panel = synthetic.rayonix_panel() if size == 3840 else synthetic.roi(synthetic.rayonix_panel(), r0, r0, size, size)
ref = np.zeros(panel.n_pixels)
p64 = SpotsPlan(synthetic.ls49_context(seed, panel=panel, compute="fp64"))
p64.run(ref, mode=N.OUT_F64)
for variant in ("3", "4"):
    os.environ["NBX_FP32_POLY"] = variant
    got = np.zeros(panel.n_pixels, dtype=np.float32)
    p32 = SpotsPlan(synthetic.ls49_context(seed, panel=panel, compute="fp32"))
    p32.run(got)
    m = parity.metrics(got, ref, panel.dims)
    m.update({"variant": f"fp32 poly deg {variant}", "size": size, "seed": seed,
              "fp64_kernel_ms": p64.kernel_ms, "fp32_kernel_ms": p32.kernel_ms})
    print(json.dumps(m), flush=True)
