import time, numpy as np, torch, ctypes
cudart = ctypes.CDLL("libcudart.so") if False else None
import torch.cuda
rt = torch.cuda.cudart()
d = torch.empty(4*1000000, dtype=torch.float64, device="cuda")
for rep in range(5):
    h = np.empty((1000000, 4))
    h[:, :] = 0  # prefault
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    r = rt.cudaHostRegister(h.ctypes.data, h.nbytes, 0)
    t1 = time.perf_counter()
    ht = torch.from_numpy(h.reshape(-1))
    ht.copy_(d, non_blocking=True); torch.cuda.synchronize()
    t2 = time.perf_counter()
    rt.cudaHostUnregister(h.ctypes.data)
    t3 = time.perf_counter()
    h2 = np.empty((1000000, 4)); h2[:, :] = 0
    t4 = time.perf_counter()
    ht2 = torch.from_numpy(h2.reshape(-1)); ht2.copy_(d); torch.cuda.synchronize()
    t5 = time.perf_counter()
    p = torch.empty(4*1000000, dtype=torch.float64).pin_memory()
    t6 = time.perf_counter(); p.copy_(d); torch.cuda.synchronize(); t7 = time.perf_counter()
    print(f"register {1e3*(t1-t0):.2f} ms, d2h registered {1e3*(t2-t1):.2f}, unregister {1e3*(t3-t2):.2f}, pageable d2h {1e3*(t5-t4):.2f}, pinned d2h {1e3*(t7-t6):.2f}  rc={r}")
