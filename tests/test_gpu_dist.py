"""The partitioned (multi-GPU) path on ONE B200: P parts of the same graph run
their sm_100a sweeps in one process and exchange slices by device copies
(dist.EmulatedExchange) -- no cross-process kernels wait on each other.  EC
must equal the oracle per 1e-12 relative with the same iteration count."""
import numpy as np
import pytest
import torch

import paper_2203_09284_b200 as fb
from paper_2203_09284_b200.dist import B200Part, partition_bounds, solve_emulated

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("P", [1, 2, 3, 4])
def test_partitioned_ec_matches_oracle(oracle, P):
    n, s, d = oracle.generate_rmat(16, 16, seed=1)
    g = oracle.build_csr(n, s, d)
    ref = oracle.pagerank_ec(g, threshold=1e-10)
    stream = fb.torch_stream_handle()
    with fb.DeviceGraph.from_graph(fb.Graph(g.n, g.m, g.in_start, g.in_src, g.out_degree)) as full:
        parts = [B200Part(full, P, r, stream=stream) for r in range(P)]
    np.testing.assert_array_equal(parts[0].bounds, partition_bounds(g.in_start, P))
    res = solve_emulated(parts, fb.ENGINE_EC, fb.PageRankConfig(threshold=1e-10))
    assert res.iterations == ref.iterations and res.converged
    assert float(np.max(np.abs(res.ranks - ref.ranks) / ref.ranks)) <= 1e-12
    fu = solve_emulated(parts, fb.ENGINE_FUSED, fb.PageRankConfig(threshold=1e-10))
    xstar = oracle.pagerank_ec(g, threshold=1e-16, max_iterations=400).ranks
    assert fu.converged and oracle.l1_norm(fu.ranks, xstar) <= g.n * 1e-10 * 0.85 / 0.15
    for p in parts:
        p.close()


@pytest.mark.parametrize("P", [2, 3, 4])
def test_fused_exchange_matches_copy_exchange(oracle, P):
    """The fused exchange (sweep epilogue stores into the other parts'
    vectors, fpr_b200_part_sweep_peers) exchanges exactly the values the copy
    all-gather would: EC is bit-identical to the copy path; FusEd (in place,
    peers see fresher values) converges within the L-inf-threshold bound."""
    n, s, d = oracle.generate_rmat(16, 16, seed=1)
    g = oracle.build_csr(n, s, d)
    stream = fb.torch_stream_handle()
    with fb.DeviceGraph.from_graph(fb.Graph(g.n, g.m, g.in_start, g.in_src, g.out_degree)) as full:
        parts = [B200Part(full, P, r, stream=stream) for r in range(P)]
    cfg = fb.PageRankConfig(threshold=1e-10)
    copy = solve_emulated(parts, fb.ENGINE_EC, cfg)
    fused = solve_emulated(parts, fb.ENGINE_EC, cfg, fused_exchange=True)
    assert fused.iterations == copy.iterations
    np.testing.assert_array_equal(fused.ranks, copy.ranks)
    assert fused.errors == copy.errors
    fu = solve_emulated(parts, fb.ENGINE_FUSED, cfg, fused_exchange=True)
    xstar = oracle.pagerank_ec(g, threshold=1e-16, max_iterations=400).ranks
    assert fu.converged and oracle.l1_norm(fu.ranks, xstar) <= g.n * 1e-10 * 0.85 / 0.15
    for p in parts:
        p.close()


def _ipc_worker(rank, world, port, path, q):
    """One of two processes on the SAME GPU: CUDA-IPC replicas + fused
    exchange, gloo for handles/pairs.  The processes' sweep kernels never wait
    on each other; the host barrier (pair all-gather) orders the iterations."""
    import os
    import sys

    sys.path.insert(0, path)
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    import torch.distributed as dist

    import paper_2203_09284_b200 as fbw
    from oracle import Oracle
    from paper_2203_09284_b200.dist import B200Part as Part, TorchExchange, solve_partitioned

    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        o = Oracle()
        n, s, d = o.generate_rmat(14, 16, seed=3)
        g = o.build_csr(n, s, d)
        with fbw.DeviceGraph.from_graph(fbw.Graph(g.n, g.m, g.in_start, g.in_src, g.out_degree)) as full:
            part = Part(full, world, rank)
        ex = TorchExchange()

        class HostGather(TorchExchange):  # gloo: slices through host memory for the one initial exchange
            def allgather_slices(self, buf, slice_):
                import torch

                h = buf.cpu()
                mine = h[self.rank * slice_:(self.rank + 1) * slice_].clone()
                self.dist.all_gather_into_tensor(h, mine)
                buf.copy_(h)

        cfg = fbw.PageRankConfig(threshold=1e-10)
        res = solve_partitioned(part, HostGather(), fbw.ENGINE_EC, cfg, fused_exchange=True, pairs_on_host=True,
                                speculate=True)
        # the same with the stop rule on the device (batches of 3 iterations
        # enqueued without a host read; sweeps past the stop are no-ops)
        dres = solve_partitioned(part, HostGather(), fbw.ENGINE_EC, cfg, fused_exchange=True, pairs_on_host=True,
                                 device_stop=True, batch=3)
        assert dres.iterations == res.iterations and dres.errors == res.errors
        assert np.array_equal(dres.ranks, res.ranks)
        # FusEd in place: peers' P2P stores land in the vector this rank is sweeping
        fres = solve_partitioned(part, HostGather(), fbw.ENGINE_FUSED, cfg, fused_exchange=True,
                                 pairs_on_host=True)
        out = [None] * world
        dist.all_gather_object(out, (res.iterations, res.ranks.tolist(), fres.converged, fres.ranks.tolist()))
        if rank == 0:
            ref = o.pagerank_ec(g, threshold=1e-10)
            xstar = o.pagerank_ec(g, threshold=1e-16, max_iterations=400).ranks
            ranks = np.concatenate([np.array(x[1]) for x in out])
            franks = np.concatenate([np.array(x[3]) for x in out])
            q.put((out[0][0], ref.iterations, float(np.max(np.abs(ranks - ref.ranks) / ref.ranks)),
                   all(x[2] for x in out), o.l1_norm(franks, xstar), g.n * 1e-10 * 0.85 / 0.15))
        part.close()
        del ex
    finally:
        dist.destroy_process_group()


def test_fused_exchange_two_processes_cuda_ipc():
    import multiprocessing as mp
    import os
    import socket

    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        port = sk.getsockname()[1]
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_ipc_worker, args=(r, 2, port, root, q)) for r in range(2)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(timeout=240)
    for p in procs:
        if p.is_alive():
            p.kill()
    assert all(p.exitcode == 0 for p in procs), [p.exitcode for p in procs]
    it, ref_it, rel, fconv, fl1, bound = q.get(timeout=5)
    assert it == ref_it and rel <= 1e-12
    assert fconv and fl1 <= bound


@pytest.mark.parametrize("P", [1, 3])
def test_part_create_matches_partition(oracle, P):
    """fpr_b200_part_create (each rank uploads only its rows) gives the same
    bounds, slice, local CSR in exchange ids and EC result as partitioning a
    full resident graph."""
    n, s, d = oracle.generate_rmat(16, 16, seed=1)
    g = oracle.build_csr(n, s, d)
    hg = fb.Graph(g.n, g.m, g.in_start, g.in_src, g.out_degree)
    stream = fb.torch_stream_handle()
    with fb.DeviceGraph.from_graph(hg) as full:
        ref_parts = [B200Part(full, P, r, stream=stream) for r in range(P)]
    parts = [B200Part.from_view(hg, P, r, stream=stream) for r in range(P)]
    for a, b in zip(parts, ref_parts):
        np.testing.assert_array_equal(a.bounds, b.bounds)
        assert a.slice == b.slice and a.n_local == b.n_local
        ga, gb = a.graph.download(), b.graph.download()
        np.testing.assert_array_equal(ga.in_start, gb.in_start)
        np.testing.assert_array_equal(ga.in_src, gb.in_src)
        np.testing.assert_array_equal(ga.out_degree, gb.out_degree)
    cfg = fb.PageRankConfig(threshold=1e-10)
    r1 = solve_emulated(parts, fb.ENGINE_EC, cfg)
    r2 = solve_emulated(ref_parts, fb.ENGINE_EC, cfg)
    assert r1.iterations == r2.iterations
    np.testing.assert_array_equal(r1.ranks, r2.ranks)
    for q in parts + ref_parts:
        q.close()

