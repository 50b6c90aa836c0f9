"""Two processes on one GPU: partitioned EC with copy exchange vs fused (IPC) exchange; print error traces."""
import os, sys
import multiprocessing as mp
import numpy as np
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def worker(rank, world, port, fused, q):
    sys.path.insert(0, ROOT)
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    import torch, torch.distributed as dist
    import paper_2203_09284_b200 as fb
    from oracle import Oracle
    from paper_2203_09284_b200.dist import B200Part, TorchExchange, solve_partitioned
    dist.init_process_group("gloo", rank=rank, world_size=world)
    o = Oracle()
    n, s, d = o.generate_rmat(14, 16, seed=3)
    g = o.build_csr(n, s, d)
    with fb.DeviceGraph.from_graph(fb.Graph(g.n, g.m, g.in_start, g.in_src, g.out_degree)) as full:
        part = B200Part(full, world, rank)

    class HostGather(TorchExchange):
        def allgather_slices(self, buf, slice_):
            h = buf.cpu()
            mine = h[self.rank * slice_:(self.rank + 1) * slice_].clone()
            self.dist.all_gather_into_tensor(h, mine)
            buf.copy_(h)

    res = solve_partitioned(part, HostGather(), fb.ENGINE_EC, fb.PageRankConfig(threshold=1e-10, max_iterations=12),
                            fused_exchange=fused, pairs_on_host=True)
    q.put((rank, fused, res.iterations, res.errors[:12]))
    dist.destroy_process_group()


if __name__ == "__main__":
    ctx = mp.get_context("spawn")
    for fused in (False, True):
        q = ctx.Queue()
        ps = [ctx.Process(target=worker, args=(r, 2, 29600 + int(fused), fused, q)) for r in range(2)]
        [p.start() for p in ps]
        [p.join(120) for p in ps]
        for _ in range(2):
            print(q.get(timeout=5), flush=True)
