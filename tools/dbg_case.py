import sys, dataclasses
sys.path.insert(0, '/root/repo/tests'); sys.path.insert(0, '/root/repo')
import numpy as np, test_gpu_fuzz as t
from oracle import oracle
from paper_2205_07976_b200 import PixelBuffer, nanobragg_spots, describe, SpotsPlan
c = t.random_case(9)
want, _ = oracle.spots(describe(c), "f64")
for shape in ("gauss", "sincg", "round", "tophat"):
    for compute in ("fp64", "fp32"):
        cc = dataclasses.replace(c, shape=shape, compute=compute)
        w, _ = oracle.spots(describe(cc), "f64")
        out = PixelBuffer.zeros(cc.panel.dims, "f64"); nanobragg_spots(cc, out)
        info = SpotsPlan(cc).info
        print(shape, compute, "variant", info.kernel_variant, "want sum %.4e got sum %.4e max %.3e nan %d" % (w.sum(), out.data.sum(), np.abs(out.data).max(), np.isnan(out.data).sum()), flush=True)
