"""Extreme shapes for the task decomposition: one hub row holding almost all
edges (split across thousands of tasks -> the cross-task partial chain at its
longest), its transpose (every row one edge), long chains of empty rows, and
rows exactly at the snap boundary.  Every engine and
the propagation-blocked EC and lockstep sweeps,
against the C oracle (EC per 1e-12 relative, same iteration count; FusEd by
the L-inf-threshold bound on L1 to x*)."""
import numpy as np
import pytest

import paper_2203_09284_b200 as fb

pytestmark = pytest.mark.gpu
EC_RTOL = 1e-12


def _csr(oracle, n, src, dst):
    g = oracle.build_csr(n, np.asarray(src, np.uint64), np.asarray(dst, np.uint64))
    return g, fb.Graph(g.n, g.m, g.in_start, g.in_src, g.out_degree)


def _shapes(oracle):
    n = (1 << 20) + 1
    others = np.arange(1, n, dtype=np.uint64)
    yield "in_star", _csr(oracle, n, others, np.zeros_like(others))            # row 0: 2^20 in-edges
    yield "out_star", _csr(oracle, n, np.zeros_like(others), others)           # 2^20 rows of 1 edge
    rng = np.random.default_rng(5)
    # two hubs + sparse background + many empty rows
    bg_s = rng.integers(0, n, 200_000).astype(np.uint64)
    bg_d = (rng.integers(0, n // 64, 200_000) * 64).astype(np.uint64)         # only every 64th row has edges
    hubs_s = rng.integers(0, n, 600_000).astype(np.uint64)
    hubs_d = np.where(rng.random(600_000) < 0.5, 7, n - 3).astype(np.uint64)  # hub rows 7 and n-3
    yield "hubs_and_gaps", _csr(oracle, n, np.concatenate([bg_s, hubs_s]), np.concatenate([bg_d, hubs_d]))
    # rows of 24..27 edges around the snap limit (25), back to back
    m_rows = 40_000
    deg = 24 + (np.arange(m_rows) % 4)
    dst = np.repeat(np.arange(m_rows, dtype=np.uint64), deg)
    src = ((np.arange(len(dst), dtype=np.uint64) * 2654435761) % m_rows).astype(np.uint64)
    yield "snap_boundary", _csr(oracle, m_rows, src, dst)


@pytest.mark.parametrize("layout", ["plain", "pb"])
def test_extreme_shapes(oracle, layout, monkeypatch):
    monkeypatch.setenv("FPR_B200_PB_CHUNK_SHIFT", "16")  # several chunks at n = 2^20
    cfg = fb.PageRankConfig(threshold=1e-10)
    for name, (g, hg) in _shapes(oracle):
        ref = oracle.pagerank_ec(g, threshold=1e-10)
        with fb.DeviceGraph.from_graph(hg, pb=layout == "pb") as dg:
            assert dg.validate() == 0
            r = dg.run(fb.ENGINE_EC, cfg)
            assert r.trace.iterations == ref.iterations, name
            assert float(np.max(np.abs(r.ranks.values - ref.ranks) / ref.ranks)) <= EC_RTOL, name
            if layout == "pb":  # the FusEd schedule on PB sweeps vs its CPU restatement
                ws = dg.wave_starts(4)
                dg.set_wave_count(4)
                lref = oracle.pagerank_lockstep(g, ws, threshold=1e-10)
                ls = dg.run(fb.ENGINE_FUSED_LOCKSTEP, cfg)
                assert ls.trace.iterations == lref.iterations, name
                assert float(np.max(np.abs(ls.ranks.values - lref.ranks) / lref.ranks)) <= EC_RTOL, name
            if layout != "plain":
                continue
            xstar = oracle.pagerank_ec(g, threshold=1e-16, max_iterations=400).ranks
            bound = g.n * 1e-10 * 0.85 / 0.15
            for eng in (fb.ENGINE_FUSED, fb.ENGINE_FUSED_LOCKSTEP):
                f = dg.run(eng, cfg)
                assert f.trace.converged, (name, eng)
                assert oracle.l1_norm(f.ranks.values, xstar) <= bound, (name, eng)


@pytest.mark.parametrize("n,edges", [
    (1, []), (2, [(0, 1), (1, 0)]), (3, [(0, 1)]), (100, []), (31, [(i, (i * 7 + 3) % 31) for i in range(31)]),
    (8192, [(i, (i * 17 + 5) % 8192) for i in range(8192)]), (8193, [(i, 8192) for i in range(8192)]),
])
def test_pb_small_and_boundary_shapes(oracle, n, edges):
    """Propagation-blocked EC and lockstep on degenerate inputs: a single
    vertex, no edges at all, fewer vertices than a warp, and n at and one
    past the 2^13-row bin boundary (the last bin holding one hub row)."""
    src = np.array([e[0] for e in edges], np.uint64)
    dst = np.array([e[1] for e in edges], np.uint64)
    g, hg = _csr(oracle, n, src, dst)
    cfg = fb.PageRankConfig(threshold=1e-10)
    ref = oracle.pagerank_ec(g, threshold=1e-10)
    with fb.DeviceGraph.from_graph(hg, pb=True) as dg:
        r = dg.run(fb.ENGINE_EC, cfg)
        assert r.trace.iterations == ref.iterations
        assert float(np.max(np.abs(r.ranks.values - ref.ranks) / ref.ranks)) <= EC_RTOL
        ws = dg.wave_starts(3)
        dg.set_wave_count(3)
        lref = oracle.pagerank_lockstep(g, ws, threshold=1e-10)
        ls = dg.run(fb.ENGINE_FUSED_LOCKSTEP, cfg)
        assert ls.trace.iterations == lref.iterations
        assert float(np.max(np.abs(ls.ranks.values - lref.ranks) / lref.ranks)) <= EC_RTOL
