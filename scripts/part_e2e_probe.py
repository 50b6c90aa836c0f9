"""Phase times of the partitioned e2e step at world size 1 (NCCL): part_create, solve, ranks, close."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import torch.distributed as dist
import paper_2203_09284_b200 as fb
from paper_2203_09284_b200.dist import B200Part, PartitionedSolver, TorchExchange

os.environ.setdefault("MASTER_ADDR", "127.0.0.1"); os.environ.setdefault("MASTER_PORT", "29533")
os.environ.setdefault("RANK", "0"); os.environ.setdefault("WORLD_SIZE", "1")
dist.init_process_group("nccl", device_id=torch.device("cuda", 0))
with fb.DeviceGraph.generate_uniform(1 << 22, 16, 2, stream=fb.torch_stream_handle()) as dg:
    g = dg.download()
def pinned(a):
    t = torch.empty(a.shape, dtype=torch.int64, pin_memory=True); v = t.numpy().view(np.uint64); v[:] = a; return t, v
keep = [pinned(g.in_start), pinned(g.in_src), pinned(g.out_degree)]
hg = fb.Graph(g.n, g.m, keep[0][1], keep[1][1], keep[2][1])
cfg = fb.PageRankConfig(threshold=1e-10)
p0 = B200Part.from_view(hg, 1, 0)
solver = PartitionedSolver(p0, TorchExchange(), device="cuda:0")
for rep in range(4):
    torch.cuda.synchronize(); t0 = time.perf_counter()
    p = B200Part.from_view(hg, 1, 0); torch.cuda.synchronize(); t1 = time.perf_counter()
    solver.rebind(p); r = solver.solve(fb.ENGINE_EC, cfg, want_ranks=False); torch.cuda.synchronize(); t2 = time.perf_counter()
    x = p.ranks(); t3 = time.perf_counter()
    p.close(); torch.cuda.synchronize(); t4 = time.perf_counter()
    print(f"create {1e3*(t1-t0):.2f} solve {1e3*(t2-t1):.2f} ({r.iterations} it) ranks {1e3*(t3-t2):.2f} close {1e3*(t4-t3):.2f} ms", flush=True)
dist.destroy_process_group()
