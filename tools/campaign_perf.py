"""Throughput of the pipelined image campaign (simulate_image + write_image per image,
run_campaign's per-rank loop) on C2 images, against the spot kernel alone.

Each image: one fused spots(+background) launch into an f64 accumulator rounded to f32, then the
download, CRC-32 and .bin write of image i overlap image i+1's kernel (nbx_campaign).
usage: python tools/campaign_perf.py [n_images] [out_dir] [--compute fp32|fp64]  (default fp64)
"""
import json
import shutil
import sys
import tempfile
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))

from paper_2205_07976_b200 import BackgroundProfile, SpotsPlan, synthetic
from paper_2205_07976_b200.io import run_campaign

compute = "fp64"
if "--compute" in sys.argv:
    i = sys.argv.index("--compute")
    compute = sys.argv[i + 1]
    del sys.argv[i:i + 2]
n = max(3, int(sys.argv[1])) if len(sys.argv) > 1 else 10
out = Path(sys.argv[2]) if len(sys.argv) > 2 else Path(tempfile.mkdtemp(prefix="nbx_campaign_"))
panel = synthetic.rayonix_panel()
water = BackgroundProfile(points=((0.0, 2.57), (0.0365, 2.58), (0.07, 2.8), (0.12, 5.0), (0.162, 8.0), (0.3, 6.5)))


def ctx_for(i):
    return synthetic.ls49_context(synthetic.SEED + i, panel=panel, compute=compute)


plan = SpotsPlan(ctx_for(0))
import torch  # noqa: E402

dev = torch.empty(plan.n_pixels, dtype=torch.float32, device="cuda")
plan.run(dev.data_ptr(), on_device=True)
kernel_ms = plan.kernel_ms
run_campaign(ctx_for, 1, out, background=water)  # warm
short = run_campaign(ctx_for, 2, out, first_image=1, background=water)
res = run_campaign(ctx_for, n, out, first_image=1, background=water)
size = sum(p.stat().st_size for p in res.paths)
print(json.dumps({"compute": compute, "images": n, "seconds": res.seconds, "images_per_s": n / res.seconds,
                  "ms_per_image": 1e3 * res.seconds / n,
                  "steady_ms_per_image": 1e3 * (res.seconds - short.seconds) / (n - 2),
                  "spot_kernel_ms": kernel_ms,
                  "bytes_written": size, "write_gbs": size / res.seconds / 1e9,
                  "note": "fused spots+background per image, f32 .bin + JSON sidecar with CRC-32, "
                          "download/CRC/write of image i overlapped with image i+1's kernel"}))
shutil.rmtree(out, ignore_errors=True)
