"""Multi-GPU host logic (paper_2203_09284_b200/dist.py) on CPU: world_size-2
gloo processes run the destination-range partition, the padded all-gather
exchange and the rank-ordered residual reduction; a numpy restatement of the
local sweep stands in for the GPU kernel.  EC must match the single-process
oracle (same iteration count, 1e-12 relative); FUSED must converge within the
geometric-tail bound."""
import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp

from paper_2203_09284_b200 import ENGINE_EC, ENGINE_FUSED, PageRankConfig
from paper_2203_09284_b200.dist import partition_bounds, remap_sources


class NumpyPart:
    """Local sweep restated with numpy (test-side checker of the host logic)."""

    def __init__(self, g, bounds, part):
        self.bounds, self.part = bounds, part
        self.slice = int(np.max(np.diff(bounds)))
        b0, b1 = int(bounds[part]), int(bounds[part + 1])
        self.n_local, self.n_global = b1 - b0, g.n
        start = g.in_start.astype(np.int64)
        self.local_start = start[b0:b1 + 1] - start[b0]
        self.src = remap_sources(g.in_src[start[b0]:start[b1]], bounds, self.slice)
        self.outdeg = g.out_degree[b0:b1].astype(np.float64)
        self.pr = None
        self.gate = None
        self.hist = []

    def init(self, exch):
        self.pr = np.full(self.n_local, 1.0 / self.n_global)
        self.hist = [self.pr]
        x = exch.numpy()
        off = self.part * self.slice
        x[off:off + self.n_local] = np.where(self.outdeg > 0, self.pr / np.maximum(self.outdeg, 1), 0.0)

    def sweep(self, engine, cfg, read, write, pair):
        if self.gate is not None and self.gate["stop"]:
            return  # gated: a stopped gate makes the sweep a no-op (fpr_b200_part_set_gate)
        rd, wr = read.numpy(), write.numpy()
        vals = rd[self.src]
        sums = np.zeros(self.n_local)
        nz = np.diff(self.local_start) > 0
        if vals.size:
            red = np.add.reduceat(vals, self.local_start[:-1][nz])
            sums[nz] = red
        nv = (1 - cfg.damping) / self.n_global + cfg.damping * sums
        d = np.abs(nv - self.pr)
        self.prev, self.pr = self.pr, nv
        off = self.part * self.slice
        wr[off:off + self.n_local] = np.where(self.outdeg > 0, nv / np.maximum(self.outdeg, 1), 0.0)
        p = pair.numpy()
        p[0], p[1] = (d.max() if d.size else 0.0), d.sum()
        self.hist.append(nv)

    # the device-side stop rule's contract (fpr_b200_gate_*), restated
    def gate_create(self, cap):
        return {"cap": cap}

    def gate_init(self, gate):
        gate.update(stop=0, iters=0, errs=[], l1s=[])

    def set_gate(self, gate):
        self.gate = gate

    def gate_update(self, gate, pairs, cfg, norm):
        if gate["stop"]:
            return
        p = pairs.numpy()
        err = max([0.0] + [float(p[2 * r]) for r in range(len(p) // 2)])
        l1 = 0.0
        for r in range(len(p) // 2):
            l1 += float(p[2 * r + 1])
        gate["errs"].append(err)
        gate["l1s"].append(l1)
        gate["iters"] += 1
        if (l1 if norm else err) <= cfg.threshold or gate["iters"] >= cfg.max_iterations:
            gate["stop"] = 1

    def gate_read(self, gate, trace=False):
        return gate["iters"], bool(gate["stop"]), list(gate["errs"]), list(gate["l1s"])

    def ranks_after(self, sweeps, out=None):
        return self.hist[sweeps]

    def ranks(self, back=0, out=None):
        r = self.prev if back else self.pr
        if out is not None:
            out[: len(r)] = r
            return out[: len(r)]
        return r


def _worker(rank, world, port, engine, threshold, out_dir, speculate=False, batch=0):
    import torch.distributed as dist

    from oracle import Oracle
    from paper_2203_09284_b200.dist import TorchExchange, solve_partitioned

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    o = Oracle()
    n, s, d = o.generate_rmat(11, 16, seed=7)
    g = o.build_csr(n, s, d)
    bounds = partition_bounds(g.in_start, world)
    local = NumpyPart(g, bounds, rank)
    res = solve_partitioned(local, TorchExchange(), engine, PageRankConfig(threshold=threshold),
                            device="cpu", speculate=speculate, device_stop=batch > 0, batch=max(batch, 1))
    np.save(os.path.join(out_dir, f"r{rank}.npy"), res.ranks)
    np.save(os.path.join(out_dir, f"e{rank}.npy"), np.array(res.errors))
    dist.destroy_process_group()


def _free_port():
    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        return sk.getsockname()[1]


def _run(engine, threshold, tmp_path, speculate=False, batch=0):
    mp.spawn(_worker, args=(2, _free_port(), engine, threshold, str(tmp_path), speculate, batch), nprocs=2,
             join=True)
    ranks = np.concatenate([np.load(tmp_path / f"r{r}.npy") for r in range(2)])
    errs = [np.load(tmp_path / f"e{r}.npy") for r in range(2)]
    return ranks, errs


def test_partition_bounds_balanced(oracle):
    n, s, d = oracle.generate_rmat(12, 16, seed=7)
    g = oracle.build_csr(n, s, d)
    for P in (1, 2, 3, 8):
        b = partition_bounds(g.in_start, P)
        assert b[0] == 0 and b[-1] == g.n and np.all(np.diff(b) >= 0)
        items = [int(g.in_start[b[r + 1]] - g.in_start[b[r]] + b[r + 1] - b[r]) for r in range(P)]
        assert max(items) - min(items) <= max(np.diff(g.in_start).max(), 1) + 1
        sl = int(np.max(np.diff(b)))
        rm = remap_sources(g.in_src, b, sl)
        part = rm // sl
        assert np.array_equal(b[part] + rm % sl, g.in_src.astype(np.int64))


@pytest.mark.parametrize("speculate", [False, True])
def test_gloo_ec_matches_oracle(oracle, tmp_path, speculate):
    """speculate=True enqueues sweep k+1 before reading iteration k's residual
    and reads the ranks one sweep back after the stop: same iteration count
    and ranks as the non-speculative driver."""
    ranks, errs = _run(ENGINE_EC, 1e-10, tmp_path, speculate)
    n, s, d = oracle.generate_rmat(11, 16, seed=7)
    ref = oracle.pagerank_ec(oracle.build_csr(n, s, d), threshold=1e-10)
    assert len(errs[0]) == len(errs[1]) == ref.iterations  # same stop decision everywhere
    assert np.array_equal(errs[0], errs[1])
    assert float(np.max(np.abs(ranks - ref.ranks) / ref.ranks)) <= 1e-12


def test_gloo_fused_converges(oracle, tmp_path):
    ranks, errs = _run(ENGINE_FUSED, 1e-10, tmp_path)
    n, s, d = oracle.generate_rmat(11, 16, seed=7)
    g = oracle.build_csr(n, s, d)
    xstar = oracle.pagerank_ec(g, threshold=1e-16, max_iterations=400).ranks
    assert errs[0][-1] <= 1e-10
    assert oracle.l1_norm(ranks, xstar) <= g.n * 1e-10 * 0.85 / 0.15


@pytest.mark.parametrize("batch", [1, 3, 8])
def test_gloo_device_stop_matches_oracle(oracle, tmp_path, batch):
    """Device-side stop (PartitionedSolver device_stop): batches of iterations
    enqueued without a host read, the gate's rule applied after each pair
    all-gather, sweeps past the stop no-ops, ranks after the stopping sweep.
    Same iteration count, trace and ranks as the host-driven loop."""
    ranks, errs = _run(ENGINE_EC, 1e-10, tmp_path, batch=batch)
    n, s, d = oracle.generate_rmat(11, 16, seed=7)
    ref = oracle.pagerank_ec(oracle.build_csr(n, s, d), threshold=1e-10)
    assert len(errs[0]) == len(errs[1]) == ref.iterations
    assert np.array_equal(errs[0], errs[1])
    assert np.allclose(errs[0], ref.errors, rtol=0, atol=1e-15)  # numpy sums vs sequential: ~1e-17 apart
    assert float(np.max(np.abs(ranks - ref.ranks) / ref.ranks)) <= 1e-12
