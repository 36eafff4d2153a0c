"""add_array on the C2 image size with device buffers (the HBM-bound helper), for ncu."""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch

from paper_2205_07976_b200 import _native as N

n = 3840 * 3840
cx = N.context()
lhs = torch.ones(n, dtype=torch.float64, device="cuda")
rhs = torch.full((n,), 0.1, dtype=torch.float32, device="cuda")
for _ in range(3):
    with cx.lock:
        N.check(cx, cx.lib.nbx_add_array(cx.handle, lhs.data_ptr(), rhs.data_ptr(), n, 1), label="add_array")
torch.cuda.synchronize()
print("add_array ok", float(lhs[0]))
