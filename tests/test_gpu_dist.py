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
