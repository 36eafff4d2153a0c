"""Where does the drop-in call spend time beyond the kernel?  (run with NBX_TRACE=1)"""
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2205_07976_b200 import PixelBuffer, describe, nanobragg_spots, synthetic

ctxs = [synthetic.ls49_context(synthetic.SEED + i, compute="fp32") for i in range(4)]
img = PixelBuffer.zeros(ctxs[0].panel.dims)
for c in ctxs:
    t0 = time.perf_counter()
    d = describe(c)
    t1 = time.perf_counter()
    nanobragg_spots(c, img)
    t2 = time.perf_counter()
    print(f"describe {1e3*(t1-t0):.1f} ms, nanobragg_spots {1e3*(t2-t1):.1f} ms", flush=True)
