"""GPU graph generation + CSR build (K5 + K4) vs the reference's
generate_rmat / random_sparse -> build_csr digests (tests/golden/), and the
config-2 EC solve on the device-built graph."""
import numpy as np
import pytest

import paper_2203_09284_b200 as fb
from golden_util import load, sha, unhex

pytestmark = pytest.mark.gpu


def digest_ok(g: fb.Graph, d: dict):
    assert g.n == d["n"] and g.m == d["m"]
    assert sha(g.in_start) == d["in_start"]
    assert sha(g.in_src) == d["in_src"]
    assert sha(g.out_degree) == d["out_degree"]
    assert int(np.diff(g.in_start).max()) == d["max_in"]


@pytest.mark.parametrize("name", ["rmat_s10_seed42.json", "rmat_s12_seed7.json", "config1.json"])
def test_rmat_generate_matches_reference(name):
    rec = load(name)
    p = rec["params"]
    with fb.DeviceGraph.generate_rmat(fb.RmatParams(p["scale"], p["edge_factor"], p["a"], p["b"],
                                                    p["c"], p["d"], p["seed"])) as dg:
        digest_ok(dg.download(), rec["graph"])


def test_rmat_golden_343():
    with fb.DeviceGraph.generate_rmat(fb.RmatParams(scale=10, edge_factor=16, seed=42)) as dg:
        assert int(dg.download().in_degree().max()) == 343


def test_generate_rejects_bad_params():
    for p in (fb.RmatParams(scale=0), fb.RmatParams(scale=33), fb.RmatParams(scale=4, edge_factor=0),
              fb.RmatParams(scale=4, edge_factor=2, a=0.9)):
        with pytest.raises(ValueError, match="rmat:"):
            fb.DeviceGraph.generate_rmat(p)


def test_config2_uniform_generate_and_ec(oracle):
    rec = load("config2.json")
    p = rec["params"]
    with fb.DeviceGraph.generate_uniform(p["n"], p["avg_degree"], p["seed"]) as dg:
        g = dg.download()
        digest_ok(g, rec["graph"])
        r = dg.run(fb.ENGINE_EC, fb.PageRankConfig(threshold=1e-10))
    run = rec["runs"]["ec_seq@1e-10"]
    assert r.trace.iterations == run["iterations"]
    assert np.max(np.abs(r.trace.errors - unhex(run["errors"]))) <= 1e-12 * float(r.ranks.values.max())
    for i, h in run["sample"].items():
        assert abs(r.ranks.values[int(i)] / float.fromhex(h) - 1) <= 1e-12
    from oracle import Graph as OGraph

    ref = oracle.pagerank_ec(OGraph(g.n, g.m, g.in_start, g.in_src, g.out_degree), threshold=1e-10)
    assert float(np.max(np.abs(r.ranks.values - ref.ranks) / ref.ranks)) <= 1e-12


# ---------------------------------------------------------------- config 3/4
def test_bfs_order_matches_oracle(oracle):
    """Device level-synchronous BFS == the sequential FIFO restatement."""
    n, s, d = oracle.generate_rmat(16, 16, seed=1)
    g = oracle.build_csr(n, s, d)
    with fb.DeviceGraph.from_graph(fb.Graph(g.n, g.m, g.in_start, g.in_src, g.out_degree)) as dg:
        for root in (0, 12345):
            np.testing.assert_array_equal(dg.bfs_order(root), oracle.bfs_relabel(g, root))


def test_rmat_relabel_generate_matches_oracle(oracle):
    n, s, d = oracle.generate_rmat(14, 16, seed=3)
    g = oracle.build_csr(n, s, d)
    want = oracle.relabel(g, oracle.bfs_relabel(g, 0))
    with fb.DeviceGraph.generate_rmat(fb.RmatParams(14, 16, seed=3), relabel_bfs=True) as dg:
        got = dg.download()
        assert dg.validate() == 0
    assert got.m == want.m == g.m
    np.testing.assert_array_equal(got.in_start, want.in_start)
    np.testing.assert_array_equal(got.in_src, want.in_src)
    np.testing.assert_array_equal(got.out_degree, want.out_degree)


def test_chunglu_generate_matches_oracle(oracle):
    n, s, d = oracle.generate_chunglu(1 << 14, 1 << 18, seed=4, kmax=10_000)
    want = oracle.build_csr(n, s, d)
    with fb.DeviceGraph.generate_chunglu(1 << 14, 1 << 18, seed=4, kmax=10_000) as dg:
        got = dg.download()
        assert dg.validate() == 0
    assert got.m == want.m
    np.testing.assert_array_equal(got.in_start, want.in_start)
    np.testing.assert_array_equal(got.in_src, want.in_src)
    np.testing.assert_array_equal(got.out_degree, want.out_degree)
