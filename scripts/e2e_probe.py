"""Breakdown of the e2e (host-buffer) path on config 2: upload/create, solve, download."""
import ctypes as C, os, sys, time
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2203_09284_b200 as fb
dg = fb.DeviceGraph.generate_uniform(1 << 22, 16, 2)
g = dg.download(); dg.close()
def pinned(a):
    t = torch.empty(a.shape, dtype=torch.int64, pin_memory=True); v = t.numpy().view(np.uint64); v[:] = a; return t, v
keep = [pinned(g.in_start), pinned(g.in_src), pinned(g.out_degree)]
pg = fb.Graph(g.n, g.m, keep[0][1], keep[1][1], keep[2][1])
cfg = fb.PageRankConfig(threshold=1e-10)
ranks = torch.empty(g.n, dtype=torch.float64, pin_memory=True)
for rep in range(4):
    t0 = time.perf_counter(); d = fb.DeviceGraph.from_graph(pg); t1 = time.perf_counter()
    r = d.run(fb.ENGINE_EC, cfg, copy_ranks=False); t15 = time.perf_counter()
    C.memmove(ranks.data_ptr(), d.ranks_device_ptr(), 8) if False else None
    t2 = time.perf_counter(); d.close(); t3 = time.perf_counter()
    print(f"  run without ranks D2H {1e3*(t15-t1):.2f} ms")
    print(f"create {1e3*(t1-t0):.2f} ms  run(+D2H ranks) {1e3*(t2-t1):.2f} ms (solve {r.solve_ms:.2f})  destroy {1e3*(t3-t2):.2f} ms")
# pageable source (std::vector-like)
pg2 = fb.Graph(g.n, g.m, g.in_start, g.in_src, g.out_degree)
for rep in range(2):
    t0 = time.perf_counter(); d = fb.DeviceGraph.from_graph(pg2); t1 = time.perf_counter(); d.close()
    print(f"pageable create {1e3*(t1-t0):.2f} ms")
x = torch.empty(604_000_000 // 8, dtype=torch.int64, pin_memory=True); y = torch.empty_like(x, device="cuda")
torch.cuda.synchronize(); t0 = time.perf_counter(); y.copy_(x); torch.cuda.synchronize(); t1 = time.perf_counter()
print(f"raw pinned H2D 604 MB: {1e3*(t1-t0):.2f} ms = {0.604/(t1-t0):.1f} GB/s")
