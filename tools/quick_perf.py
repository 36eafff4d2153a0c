"""Quick device-time probe of the spot kernel on the C2 (LS49-shape) workload."""
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch

from paper_2205_07976_b200 import SpotsPlan, synthetic
from paper_2205_07976_b200 import _native as N

size = int(sys.argv[1]) if len(sys.argv) > 1 else 3840
for compute in sys.argv[2:] or ["fp32", "fp64"]:
    t0 = time.time()
    panel = synthetic.roi(synthetic.rayonix_panel(), (3840 - size) // 2, (3840 - size) // 2, size, size)
    ctx = synthetic.ls49_context(panel=panel, compute=compute)
    plan = SpotsPlan(ctx)
    t1 = time.time()
    out = torch.empty(plan.n_pixels, dtype=torch.float32, device="cuda")
    for i in range(3):
        plan.run(out.data_ptr(), mode=N.OUT_F32, on_device=True)
        ms = plan.kernel_ms
        print(f"{compute} {size}^2: plan {t1-t0:.2f}s kernel {ms:.1f} ms  {plan.steps/ms/1e6:.1f} Gsteps/s "
              f"table {list(plan.info.table_dim)} kind {plan.info.table_kind}", flush=True)
