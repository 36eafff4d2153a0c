"""FP64 path: time the spot kernel of several builds of libnbx.so on the full C2 image and
compare their images (kernel experiments: each build differs by -D switches).

usage: python tools/fp64_variants.py [--size N] [--runs R] name=path/to/libnbx.so [name=path ...]
       (a bare `name=` uses the in-tree library)
Each build runs in its own process (NBX_LIB selects the library); the first build's image is the
reference the others are compared with (tests/parity.py metrics: total, per spot, per pixel).
"""
import json
import os
import subprocess
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]


def child(size: int, runs: int, out: str) -> None:
    sys.path.insert(0, str(ROOT))
    import numpy as np
    import torch

    from paper_2205_07976_b200 import SpotsPlan, synthetic
    from paper_2205_07976_b200 import _native as N

    r0 = (3840 - size) // 2
    panel = synthetic.rayonix_panel() if size == 3840 else synthetic.roi(synthetic.rayonix_panel(), r0, r0, size, size)
    ctx = synthetic.ls49_context(panel=panel, compute="fp64")
    p = SpotsPlan(ctx)
    img = torch.empty(p.n_pixels, dtype=torch.float64, device="cuda")
    ms = []
    for _ in range(runs):
        p.run(img.data_ptr(), mode=N.OUT_F64, on_device=True)
        ms.append(p.kernel_ms)
    np.save(out, img.cpu().numpy().reshape(panel.dims))
    print(json.dumps({"ms": ms, "best_ms": min(ms), "gsteps": p.steps / min(ms) / 1e6,
                      "variant": p.info.kernel_variant}))


def main() -> None:
    args = sys.argv[1:]
    size, runs = 3840, 3
    if "--size" in args:
        i = args.index("--size"); size = int(args[i + 1]); del args[i:i + 2]
    if "--runs" in args:
        i = args.index("--runs"); runs = int(args[i + 1]); del args[i:i + 2]
    sys.path.insert(0, str(ROOT / "tests"))
    sys.path.insert(0, str(ROOT))
    import numpy as np

    results = {}
    for spec in args:
        name, _, lib = spec.partition("=")
        env = dict(os.environ)
        if lib:
            env["NBX_LIB"] = str(Path(lib).resolve())
        out = f"/tmp/fp64v_{name}.npy"
        r = subprocess.run([sys.executable, __file__, "--child", str(size), str(runs), out], env=env,
                           capture_output=True, text=True)
        if r.returncode != 0:
            print(f"{name}: FAILED\n{r.stderr[-2000:]}", flush=True)
            continue
        res = json.loads(r.stdout.strip().splitlines()[-1])
        results[name] = (res, np.load(out))
        print(f"{name}: {[round(m, 2) for m in res['ms']]} ms, {res['gsteps']:.1f} Gsteps/s "
              f"(variant {res['variant']})", flush=True)
    if len(results) > 1:
        import parity

        names = list(results)
        ref = results[names[0]][1]
        for n in names[1:]:
            m = parity.metrics(results[n][1], ref, ref.shape)
            print(f"{n} vs {names[0]}: total {m['total']:.2e} spot {m['spot']:.2e} "
                  f"pixabs/max {m['pix_abs_over_max']:.2e}", flush=True)


if __name__ == "__main__":
    if len(sys.argv) > 1 and sys.argv[1] == "--child":
        child(int(sys.argv[2]), int(sys.argv[3]), sys.argv[4])
    else:
        main()
