import time, numpy as np, torch, ctypes, threading
from concurrent.futures import ThreadPoolExecutor
cr = torch.cuda.cudart()
n = 8 << 30
a = np.ones(n // 8)
t=time.perf_counter(); r = cr.cudaHostRegister(a.ctypes.data, a.nbytes, 0); t1=time.perf_counter()
print("register 8GB", r, f"{t1-t:.3f}s -> {a.nbytes/(t1-t)/1e9:.1f} GB/s")
t=time.perf_counter(); cr.cudaHostUnregister(a.ctypes.data); print("unregister", time.perf_counter()-t)
# readonly flag = 8
t=time.perf_counter(); r = cr.cudaHostRegister(a.ctypes.data, a.nbytes, 8); t1=time.perf_counter()
print("register RO", r, f"{t1-t:.3f}s"); cr.cudaHostUnregister(a.ctypes.data)
# multithreaded memcpy pageable -> pinned
p = torch.empty(n // 8, dtype=torch.float64, pin_memory=True).numpy()
p[:] = 0
for th in (1, 4, 8, 16):
    chunks = np.array_split(np.arange(a.size), th*4)
    def cp(idx):
        s, e = idx[0], idx[-1]+1
        np.copyto(p[s:e], a[s:e])
    with ThreadPoolExecutor(th) as ex:
        t=time.perf_counter(); list(ex.map(cp, chunks)); dt=time.perf_counter()-t
    print(f"memcpy threads {th}: {a.nbytes/dt/1e9:.1f} GB/s")
# H2D from pageable
d = torch.empty(n//8, dtype=torch.float64, device='cuda')
ta = torch.from_numpy(a)
for _ in range(2):
    torch.cuda.synchronize(); t=time.perf_counter(); d.copy_(ta); torch.cuda.synchronize(); print(f"H2D pageable {a.nbytes/(time.perf_counter()-t)/1e9:.1f} GB/s")
tp = torch.from_numpy(p)
torch.cuda.synchronize(); t=time.perf_counter(); d.copy_(tp); torch.cuda.synchronize(); print(f"H2D pinned {a.nbytes/(time.perf_counter()-t)/1e9:.1f} GB/s")
