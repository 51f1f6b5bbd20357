import ctypes as C, time, numpy as np
cudart = C.CDLL("libcudart.so") if False else None
import torch
torch.cuda.init()
lib = C.CDLL(torch._C.__file__) if False else None
# use cuda-python-free path: torch.cuda.cudart()
cr = torch.cuda.cudart()
for mb in (64, 256, 829):
    a = np.ones(mb << 20, np.uint8)
    t = time.perf_counter()
    r = cr.cudaHostRegister(a.ctypes.data, a.nbytes, 0)
    t1 = time.perf_counter() - t
    t = time.perf_counter()
    cr.cudaHostUnregister(a.ctypes.data)
    t2 = time.perf_counter() - t
    print(f"{mb} MB: register {t1*1e3:.1f} ms ({mb/1024/t1:.1f} GB/s), unregister {t2*1e3:.1f} ms, rc={r}")
