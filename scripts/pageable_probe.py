"""Pageable host -> device upload options for 604 MB (config 2's u64 CSR)."""
import time, threading
import numpy as np, torch
n = 604_000_000 // 8
a = np.random.randint(0, 1 << 22, size=n, dtype=np.uint64)   # pageable, touched
d = torch.empty(n, dtype=torch.int64, device="cuda")
cudart = torch.cuda.cudart()
for rep in range(2):
    torch.cuda.synchronize(); t0 = time.perf_counter()
    d.copy_(torch.from_numpy(a.view(np.int64)), non_blocking=False); torch.cuda.synchronize()
    t1 = time.perf_counter(); print(f"driver pageable copy: {1e3*(t1-t0):.1f} ms")
for rep in range(2):
    t0 = time.perf_counter()
    r = cudart.cudaHostRegister(a.ctypes.data, a.nbytes, 0)
    t1 = time.perf_counter()
    d.copy_(torch.from_numpy(a.view(np.int64)), non_blocking=True); torch.cuda.synchronize()
    t2 = time.perf_counter()
    cudart.cudaHostUnregister(a.ctypes.data); t3 = time.perf_counter()
    print(f"register {1e3*(t1-t0):.1f} ms + copy {1e3*(t2-t1):.1f} ms + unregister {1e3*(t3-t2):.1f} ms (rc {r})")
# threaded staging into pinned ring
CH = 8 << 20  # elements per chunk (64 MB)
stage = [torch.empty(CH, dtype=torch.int64, pin_memory=True) for _ in range(3)]
sv = [s.numpy() for s in stage]
s_copy = torch.cuda.Stream()
def staged(nthreads):
    ev = [None] * 3
    av = a.view(np.int64)
    t0 = time.perf_counter()
    for i, off in enumerate(range(0, n, CH)):
        k = i % 3; cnt = min(CH, n - off)
        if ev[k] is not None: ev[k].synchronize()
        per = (cnt + nthreads - 1) // nthreads
        ths = [threading.Thread(target=lambda j=j: np.copyto(sv[k][j*per:min(cnt,(j+1)*per)], av[off+j*per:off+min(cnt,(j+1)*per)])) for j in range(nthreads)]
        [t.start() for t in ths]; [t.join() for t in ths]
        with torch.cuda.stream(s_copy):
            d[off:off+cnt].copy_(stage[k][:cnt], non_blocking=True)
            ev[k] = torch.cuda.Event(); ev[k].record(s_copy)
    torch.cuda.synchronize()
    return time.perf_counter() - t0
import os
for nt in (1, 4, 8, 16):
    print(f"staged {nt} threads: {1e3*staged(nt):.1f} ms  (cpus {os.cpu_count()})")
