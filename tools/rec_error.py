"""FP64 channel-recurrence variants vs the direct FP64 kernel on LS49 ROIs, and their C2 kernel time.

    python tools/rec_error.py [--full | --full-only]

Variants (NBX_FP64_REC): unset = segmented recurrence (kernel_variant 6, the default),
1 = per-channel bracket recurrence (4), 0 = direct per-channel evaluation (0, the reference
for the accuracy columns).  --full also times the whole C2 image with each variant.
"""
import os
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
sys.path.insert(0, str(Path(__file__).resolve().parents[1] / "tests"))
import numpy as np

import parity
from paper_2205_07976_b200 import SpotsPlan, synthetic
from paper_2205_07976_b200 import _native as N

VARIANTS = {"segmented": None, "bracket": "1"}


def run(ctx, rec):
    if rec is None:
        os.environ.pop("NBX_FP64_REC", None)
    else:
        os.environ["NBX_FP64_REC"] = rec
    p = SpotsPlan(ctx)
    out = np.zeros(p.n_pixels)
    p.run(out, mode=N.OUT_F64)
    info = p.info
    res = out, p.kernel_ms, info.kernel_variant
    p.close()
    return res


for seed in (() if "--full-only" in sys.argv else (0, 1, 2)):
    for r0 in (1888, 600, 40):
        panel = synthetic.roi(synthetic.rayonix_panel(), r0, r0, 128, 128)
        ctx = synthetic.ls49_context(synthetic.SEED + seed, panel=panel, compute="fp64")
        direct, kd, _ = run(ctx, "0")
        for name, rec in VARIANTS.items():
            got, k, v = run(ctx, rec)
            m = parity.metrics(got, direct, panel.dims)
            print(f"seed {seed} r0 {r0} {name:9s} (variant {v}): total {m['total']:.2e} spot {m['spot']:.2e} "
                  f"pixabs/max {m['pix_abs_over_max']:.2e} pixrel(bright) {m['pix_rel_bright']:.2e}  "
                  f"{k:.2f} ms (direct {kd:.2f} ms)", flush=True)

if "--full" in sys.argv or "--full-only" in sys.argv:
    ctx = synthetic.ls49_context(synthetic.SEED, compute="fp64")
    for name, rec in VARIANTS.items():
        os.environ.pop("NBX_FP64_REC", None) if rec is None else os.environ.__setitem__("NBX_FP64_REC", rec)
        p = SpotsPlan(ctx)
        import torch

        out = torch.empty(p.n_pixels, dtype=torch.float32, device="cuda")
        ms = []
        for _ in range(3):
            p.run(out.data_ptr(), mode=N.OUT_F32, on_device=True)
            ms.append(p.kernel_ms)
        print(f"C2 full {name} (variant {p.info.kernel_variant}): {ms} ms, "
              f"{p.steps / min(ms) / 1e6:.1f} Gsteps/s", flush=True)
        p.close()
