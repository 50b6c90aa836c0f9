"""Pinned-upload split sweep: share of in_src narrowed by host threads (FPR_B200_HOST_NARROW)
vs raw DMA + device narrowing; config 2 graph_create time and full fpr_b200_pagerank e2e."""
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
print("host threads:", os.cpu_count(), "omp:", os.environ.get("OMP_NUM_THREADS"))
ref = None
for share in [float(x) for x in (sys.argv[1:] or "0 0.5 0.6 0.7 0.8 0.9 1".split())]:
    os.environ["FPR_B200_HOST_NARROW"] = str(share)
    ts = []
    for rep in range(5):
        torch.cuda.synchronize(); t0 = time.perf_counter(); d = fb.DeviceGraph.from_graph(pg)
        torch.cuda.synchronize(); ts.append(time.perf_counter() - t0)
        if rep == 4:
            x = d.download()
            assert np.array_equal(x.in_src, g.in_src) and np.array_equal(x.out_degree, g.out_degree)
        d.close()
    print(f"share {share:.2f}: create min {1e3*min(ts):.2f} ms median {1e3*sorted(ts)[2]:.2f} ms", flush=True)
