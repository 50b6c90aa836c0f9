"""fpr_b200_graph_from_edges = fpr::build_csr(EdgeSet) on the device, checked
the way the reference's graph_core_test.cpp checks build_csr (:38-98), on the
200-graph golden corpus, and on config 2's 2^26 draws (pinned and pageable
uploads) against the reference's CSR digests."""
import numpy as np
import pytest

import paper_2203_09284_b200 as fb
from golden_util import load, sha

pytestmark = pytest.mark.gpu


def _build(n, edges):
    e = np.array(edges, np.uint64).reshape(-1, 2)
    return fb.build_csr(n, e[:, 0], e[:, 1])


def test_three_sources_one_sink():
    g = _build(4, [(0, 3), (1, 3), (2, 3)])
    assert (g.n, g.m) == (4, 3)
    assert g.in_start.tolist() == [0, 0, 0, 0, 3]
    assert g.in_src.tolist() == [0, 1, 2]
    assert g.out_degree.tolist() == [1, 1, 1, 0]


def test_drops_duplicates_and_self_loops():
    g = _build(2, [(0, 1), (0, 1), (1, 1)])
    assert g.m == 1 and g.in_src.tolist() == [0] and g.out_degree.tolist() == [1, 0]


def test_empty_graph():
    g = _build(1, [])
    assert g.in_start.tolist() == [0, 0] and g.m == 0 and g.out_degree.tolist() == [0]


def test_rejects_out_of_range_vertex():
    with pytest.raises(ValueError) as ei:
        _build(2, [(0, 1), (0, 2)])
    assert str(ei.value) == "build_csr: edge #1 (0,2) has endpoint outside [0,2)"


def test_in_segments_sorted_ascending():
    assert _build(5, [(4, 0), (2, 0), (3, 0), (1, 0)]).in_src.tolist() == [1, 2, 3, 4]


def test_idempotent_on_normalized_input():
    rng = np.random.default_rng(11)
    for _ in range(20):
        n = int(rng.integers(1, 31))
        mask = rng.random((n, n)) < 0.3
        src, dst = np.nonzero(mask)
        g1 = fb.build_csr(n, src, dst)
        dst1 = np.repeat(np.arange(n, dtype=np.uint64), np.diff(g1.in_start.astype(np.int64)))
        g2 = fb.build_csr(n, g1.in_src, dst1)
        for a in ("in_start", "in_src", "out_degree"):
            np.testing.assert_array_equal(getattr(g1, a), getattr(g2, a))


def test_golden_corpus_matches_oracle(oracle):
    for rec in load("corpus.json"):
        e = np.array(rec["edges"], np.uint64).reshape(-1, 2)
        want = oracle.build_csr(rec["n"], e[:, 0], e[:, 1])
        got = fb.build_csr(rec["n"], e[:, 0], e[:, 1])
        assert got.m == want.m
        np.testing.assert_array_equal(got.in_start, want.in_start)
        np.testing.assert_array_equal(got.in_src, want.in_src)
        np.testing.assert_array_equal(got.out_degree, want.out_degree)


@pytest.mark.parametrize("pinned", [False, True])
def test_config2_draws_digest(oracle, pinned):
    import torch

    rec = load("config2.json")
    n, s, d = oracle.random_sparse(rec["params"]["n"], rec["params"]["avg_degree"], rec["params"]["seed"])
    assert sha(s) == rec["draws_sha256"]["src"] and sha(d) == rec["draws_sha256"]["dst"]
    if pinned:
        ts = torch.empty(len(s), dtype=torch.int64, pin_memory=True)
        td = torch.empty(len(d), dtype=torch.int64, pin_memory=True)
        ts.numpy().view(np.uint64)[:] = s
        td.numpy().view(np.uint64)[:] = d
        s, d = ts.numpy().view(np.uint64), td.numpy().view(np.uint64)
    with fb.DeviceGraph.from_edges(n, s, d) as dg:
        g = dg.download()
        r = dg.run(fb.ENGINE_EC, fb.PageRankConfig(threshold=1e-10), copy_ranks=False)
    gd = rec["graph"]
    assert (g.n, g.m) == (gd["n"], gd["m"])
    assert sha(g.in_start) == gd["in_start"] and sha(g.in_src) == gd["in_src"]
    assert sha(g.out_degree) == gd["out_degree"]
    assert r.trace.iterations == rec["runs"]["ec_seq@1e-10"]["iterations"]
