"""How well is an FP64 image determined by its FP64 inputs?  Runs the REFERENCE itself
(xtrace.kernels.nanobragg_spots, /root/reference; this container only) on a golden fixture twice more
with every fractional Miller index h perturbed by one ulp (up, then down) inside its grating
function (kernels.py:134-142), and reports the relative change of the total, the spots and the
bright pixels against the unperturbed reference image.  Any FP64 implementation rounds h (and pi h,
N pi h) somewhere, so differences of this size between two correct FP64 implementations are
expected; on ls49_edge (|h| ~ 35, N = 30) the bright pixels next to an exact Bragg condition move by
~1e-8 -- the 6e-9 per-pixel difference between this package's FP64 path and the reference there
(profiles/*_parity.json, pix_rel_bright), while total and spots agree to ~1e-12.

usage: python tools/conditioning.py [fixture ...]   (default: ls49_edge ls49_centre)
"""
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT / "tools"))
sys.path.insert(0, str(ROOT / "tests"))
import numpy as np

import make_golden  # imports the reference from /root/reference/pkg/src
import parity

xk = make_golden.xk


def run(case, ulps):
    real = xk._sincg_grid

    def nudged(t, n):
        u = t
        for _ in range(abs(ulps)):
            u = np.nextafter(u, np.inf if ulps > 0 else -np.inf)
        return real(u, n)

    xk._sincg_grid = nudged
    try:
        return make_golden.run_reference(case)[1]
    finally:
        xk._sincg_grid = real


def main(names):
    for name in names:
        case = parity.load(name)
        dims = (int(case["panel"][0]), int(case["panel"][1]))
        ref = case["ref_f64"]
        for ulps in (1, -1):
            img = run(case, ulps)
            m = parity.metrics(img, ref, dims)
            print(f"{name}: h {ulps:+d} ulp -> total {m['total']:.1e} spot {m['spot']:.1e} "
                  f"pixabs/max {m['pix_abs_over_max']:.1e} pixrel(bright) {m['pix_rel_bright']:.1e}", flush=True)


if __name__ == "__main__":
    main(sys.argv[1:] or ["ls49_edge", "ls49_centre"])
