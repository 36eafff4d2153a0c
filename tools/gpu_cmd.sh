mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_gpu.log
timeout 300 python tools/rec_error.py --full-only > gpurun_out/rec_error.log 2>&1
cat > /tmp/noise_probe.py <<'PY'
import sys; sys.path.insert(0, '.')
import numpy as np, torch
from paper_2205_07976_b200 import _native as N
cx = N.context()
n = 3840 * 3840
mean = (torch.rand(n, dtype=torch.float32, device="cuda") * 100)
out = torch.empty_like(mean)
for _ in range(3):
    assert cx.lib.nbx_add_noise(cx.handle, N.C.c_void_p(mean.data_ptr()), N.C.c_void_p(out.data_ptr()), n, 0, 7, 0, 1) == 0
torch.cuda.synchronize()
PY
timeout 600 ncu --set full --clock-control none --import-source on -k regex:noise_kernel -s 1 -c 1 -o gpurun_out/noise -f python /tmp/noise_probe.py > gpurun_out/ncu_noise.log 2>&1; echo "rc=$?" >> gpurun_out/ncu_noise.log
tail -5 gpurun_out/pytest_gpu.log; cat gpurun_out/rec_error.log; tail -2 gpurun_out/ncu_noise.log
