import sys, dataclasses, os
sys.path.insert(0, '/root/repo'); sys.path.insert(0, '/root/repo/tests')
import numpy as np, parity
from paper_2205_07976_b200 import SpotsPlan, synthetic
from paper_2205_07976_b200 import _native as N
for n in (30, 60, 100, 150):
    for r0 in (1888, 600):
        panel = synthetic.roi(synthetic.rayonix_panel(), r0, r0, 128, 128)
        ctx = synthetic.ls49_context(panel=panel)
        ctx = dataclasses.replace(ctx, crystal=dataclasses.replace(ctx.crystal, n_cells=(n, n, n)))
        ref = np.zeros(panel.n_pixels); SpotsPlan(dataclasses.replace(ctx, compute="fp64")).run(ref, mode=N.OUT_F64)
        out = {}
        for num in ("mufu", "poly"):
            os.environ["NBX_FP32_NUM"] = num
            got = np.zeros(panel.n_pixels); SpotsPlan(dataclasses.replace(ctx, compute="fp32")).run(got, mode=N.OUT_F64)
            m = parity.metrics(got, ref, panel.dims); out[num] = (m['total'], m['spot'], m['n_spots'])
        print(n, r0, "mufu total %.2e spot %.2e (%d)" % out["mufu"], "| poly total %.2e spot %.2e" % out["poly"][:2], flush=True)
