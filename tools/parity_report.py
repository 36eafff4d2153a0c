"""Parity margins of both compute paths on every golden fixture (reference-run outputs).

Prints one JSON object per (case, path): relative error of the total and of the worst
spot, per-pixel diagnostics, and the tolerance the tests assert (FP64 1e-9, FP32 1e-4).
usage: python tools/parity_report.py [> profiles/<round>_parity.json]
"""
import json
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "tests"))

import parity  # noqa: E402
from paper_2205_07976_b200 import PixelBuffer, nanobragg_spots  # noqa: E402

CASES = ["thomson", "scalar_match", "triclinic_pol_2wl", "pipeline_spots", "c1_toy", "tilted", "ls49_centre",
         "ls49_edge"]
TOL = {"fp64": 1e-9, "fp32": 1e-4}

rows = []
for name in CASES:
    case = parity.load(name)
    dims = (int(case["panel"][0]), int(case["panel"][1]))
    for compute in ("fp64", "fp32"):
        out = PixelBuffer.zeros(dims, "f64" if compute == "fp64" else "f32")
        nanobragg_spots(parity.context(case, compute), out)
        m = parity.metrics(out.data, case["ref_f64"], dims)
        m.update({"case": name, "path": compute, "tol": TOL[compute],
                  "margin": TOL[compute] / max(m["total"], m["spot"], 1e-300)})
        rows.append(m)
        print(json.dumps(m), flush=True)
worst = {c: min(r["margin"] for r in rows if r["path"] == c) for c in TOL}
print(json.dumps({"summary": "smallest tolerance/error margin over all cases", **worst}))
