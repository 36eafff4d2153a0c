import sys; sys.path.insert(0,'/root/repo')
import torch
from paper_2205_07976_b200 import _native as N
cx=N.context(0); lib,h=cx.lib,cx.handle
n=3840*3840
f32=torch.rand(n,dtype=torch.float32,device='cuda')*100
four=(N.C.c_double*4)(); counts=(N.C.c_int64*64)(); uo,oo=N.C.c_int64(0),N.C.c_int64(0)
for _ in range(3):
    lib.nbx_image_stats(h, N.C.c_void_p(f32.data_ptr()), n, 0, 1, four)
    lib.nbx_image_histogram(h, N.C.c_void_p(f32.data_ptr()), n, 0, 1, 64, 0.0, 100.0, counts, N.C.byref(uo), N.C.byref(oo))
torch.cuda.synchronize(); print('ok')
out32 = torch.empty(n, dtype=torch.float32, device='cuda')
for _ in range(3):
    lib.nbx_add_noise(h, N.C.c_void_p(f32.data_ptr()), N.C.c_void_p(out32.data_ptr()), n, 0, 7, 0, 1)
torch.cuda.synchronize(); print('noise ok')
