"""FP64 channel recurrence vs the direct FP64 kernel on LS49 ROIs (accuracy of the recurrence)."""
import os
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
sys.path.insert(0, str(Path(__file__).resolve().parents[1] / "tests"))
import numpy as np

import parity
from paper_2205_07976_b200 import SpotsPlan, synthetic
from paper_2205_07976_b200 import _native as N

for seed in (0, 1, 2):
    for r0 in (1888, 600, 40):
        panel = synthetic.roi(synthetic.rayonix_panel(), r0, r0, 128, 128)
        ctx = synthetic.ls49_context(synthetic.SEED + seed, panel=panel, compute="fp64")
        os.environ.pop("NBX_FP64_REC", None)
        p = SpotsPlan(ctx)
        rec = np.zeros(p.n_pixels)
        p.run(rec, mode=N.OUT_F64)
        krec = p.kernel_ms
        os.environ["NBX_FP64_REC"] = "0"
        q = SpotsPlan(ctx)
        direct = np.zeros(q.n_pixels)
        q.run(direct, mode=N.OUT_F64)
        m = parity.metrics(rec, direct, panel.dims)
        print(f"seed {seed} r0 {r0}: total {m['total']:.2e} spot {m['spot']:.2e} pixabs/max {m['pix_abs_over_max']:.2e} "
              f"pixrel(bright) {m['pix_rel_bright']:.2e}  rec {krec:.2f} ms direct {q.kernel_ms:.2f} ms", flush=True)
