"""Pin the C restatement (oracle/fpr_oracle.c) against the reference's own
outputs (tests/golden/, produced by tests/golden/make_golden.py from the
unmodified reference).  CPU only.  Bit-exact: the restatement must reproduce
the reference's bytes, not approximate them."""
import hashlib

import numpy as np
import pytest

from golden_util import load, sha, small_edges, unhex
from oracle import NORM_L1


def _graph_matches(g, digest):
    assert g.n == digest["n"] and g.m == digest["m"]
    assert sha(g.in_start) == digest["in_start"]
    assert sha(g.in_src) == digest["in_src"]
    assert sha(g.out_degree) == digest["out_degree"]
    assert int(np.diff(g.in_start).max()) == digest["max_in"]


def _run_matches(r, digest):
    assert r.iterations == digest["iterations"]
    np.testing.assert_array_equal(r.errors, unhex(digest["errors"]))
    assert sha(r.ranks) == digest["ranks_sha256"]
    for i, h in digest["sample"].items():
        assert r.ranks[int(i)] == float.fromhex(h)


def test_kats(oracle):
    """SPEC.md:208-221 examples as produced by the reference."""
    for name, rec in load("kat.json").items():
        g = oracle.build_csr(*small_edges(rec))
        assert g.m == rec["m"], name
        assert g.in_start.tolist() == rec["in_start"]
        assert g.in_src.tolist() == rec["in_src"]
        assert g.out_degree.tolist() == rec["out_degree"]
        ec = oracle.pagerank_ec(g, threshold=1e-15)
        assert ec.iterations == rec["ec_seq"]["iterations"], name
        np.testing.assert_array_equal(ec.ranks, unhex(rec["ec_seq"]["ranks"]))
        np.testing.assert_array_equal(ec.errors, unhex(rec["ec_seq"]["errors"]))
        fu = oracle.pagerank_fused_seq(g, threshold=1e-15)
        assert fu.iterations == rec["fused_seq"]["iterations"], name
        np.testing.assert_array_equal(fu.ranks, unhex(rec["fused_seq"]["ranks"]))
        one = oracle.pagerank_ec(g, threshold=1e-15, max_iterations=1)
        np.testing.assert_array_equal(one.ranks, unhex(rec["ec_one_step"]))
        np.testing.assert_array_equal(oracle.dense_oracle(g, threshold=1e-15), unhex(rec["dense"]))


def test_spec_examples_literal(oracle):
    """The literal SPEC values (independent of the fixtures)."""
    g = oracle.build_csr(2, np.array([0, 1], np.uint64), np.array([1, 0], np.uint64))
    r = oracle.pagerank_ec(g, threshold=1e-15)
    assert r.iterations == 1 and r.ranks.tolist() == [0.5, 0.5]
    g = oracle.build_csr(1, np.zeros(0, np.uint64), np.zeros(0, np.uint64))
    r = oracle.pagerank_ec(g, threshold=1e-15)
    assert r.iterations == 2 and r.ranks[0] == pytest.approx(0.15, abs=1e-16)
    g = oracle.build_csr(3, np.array([0, 1, 2, 2], np.uint64), np.array([2, 2, 0, 1], np.uint64))
    r = oracle.pagerank_ec(g, threshold=1e-15, max_iterations=1)
    np.testing.assert_allclose(r.ranks, [0.05 + 0.85 / 6, 0.05 + 0.85 / 6, 0.05 + 0.85 * 2 / 3], rtol=1e-15)


def test_corpus(oracle):
    """SPEC AC1/AC2 corpus: bit-exact vs reference ec_seq / fused_seq / dense."""
    for rec in load("corpus.json"):
        g = oracle.build_csr(*small_edges(rec))
        ec = oracle.pagerank_ec(g, threshold=1e-13)
        assert ec.iterations == rec["ec_seq"]["iterations"]
        np.testing.assert_array_equal(ec.ranks, unhex(rec["ec_seq"]["ranks"]))
        fu = oracle.pagerank_fused_seq(g, threshold=1e-13)
        assert fu.iterations == rec["fused_seq"]["iterations"]
        np.testing.assert_array_equal(fu.ranks, unhex(rec["fused_seq"]["ranks"]))
        np.testing.assert_array_equal(oracle.dense_oracle(g, threshold=1e-13), unhex(rec["dense"]))
        # AC1: ec_seq vs dense oracle within L-inf 1e-9.
        assert oracle.linf_norm(ec.ranks, unhex(rec["dense"])) <= 1e-9


@pytest.mark.parametrize("name", ["rmat_s10_seed42.json", "rmat_s12_seed7.json", "config1.json"])
def test_rmat_graphs(oracle, name):
    rec = load(name)
    p = rec["params"]
    n, s, d = oracle.generate_rmat(p["scale"], p["edge_factor"], p["a"], p["b"], p["c"], p["d"], p["seed"])
    assert sha(s) == rec["draws_sha256"]["src"] and sha(d) == rec["draws_sha256"]["dst"]
    g = oracle.build_csr(n, s, d)
    _graph_matches(g, rec["graph"])
    for key, dig in rec["runs"].items():
        eng, t = key.split("@")
        fn = oracle.pagerank_ec if eng == "ec_seq" else oracle.pagerank_fused_seq
        _run_matches(fn(g, threshold=float(t)), dig)


@pytest.mark.parametrize("name", ["rmat_s12_seed7.json", "config1.json"])
def test_ec_step_chain_is_the_reference_run(oracle, name):
    """fo_ec_step (OpenMP over rows) chained from 1/n reproduces the
    reference's ec_seq run bit for bit: the same ranks hash, iteration count
    and max-delta trace as the golden fixture.  The full-size one-step GPU
    checks (tests/test_gpu_fullsize.py) rest on this."""
    rec = load(name)
    p = rec["params"]
    g = oracle.build_csr(*oracle.generate_rmat(p["scale"], p["edge_factor"], p["a"], p["b"], p["c"], p["d"],
                                               p["seed"]))
    dig = rec["runs"]["ec_seq@1e-10"]
    x = np.full(g.n, 1.0 / g.n)
    errs = []
    for _ in range(dig["iterations"]):
        x, err, _l1 = oracle.ec_step(g, x)
        errs.append(err)
    assert [e.hex() for e in errs] == dig["errors"]
    assert sha(x) == dig["ranks_sha256"]


def test_rmat_golden_343(oracle):
    """io_ingest_test.cpp:143-155: max in-degree 343 at scale 10, ef 16, seed 42."""
    n, s, d = oracle.generate_rmat(10, 16, seed=42)
    g = oracle.build_csr(n, s, d)
    assert int(g.in_degree().max()) == 343


def test_lockstep_degenerate_cases(oracle):
    """One wave == EC exactly; one vertex per wave == fused_seq exactly."""
    n, s, d = oracle.generate_rmat(10, 16, seed=42)
    g = oracle.build_csr(n, s, d)
    ec = oracle.pagerank_ec(g, threshold=1e-12)
    ls1 = oracle.pagerank_lockstep(g, np.array([0, n], np.uint64), threshold=1e-12)
    assert ls1.iterations == ec.iterations
    np.testing.assert_array_equal(ls1.ranks, ec.ranks)
    fu = oracle.pagerank_fused_seq(g, threshold=1e-12)
    lsn = oracle.pagerank_lockstep(g, np.arange(n + 1, dtype=np.uint64), threshold=1e-12)
    assert lsn.iterations == fu.iterations
    np.testing.assert_array_equal(lsn.ranks, fu.ranks)


def test_l1_norm_mode(oracle):
    """The L1 stop rule (BASELINE wording) takes more iterations than L-inf."""
    n, s, d = oracle.generate_rmat(12, 16, seed=7)
    g = oracle.build_csr(n, s, d)
    a = oracle.pagerank_ec(g, threshold=1e-10)
    b = oracle.pagerank_ec(g, threshold=1e-10, norm=NORM_L1)
    assert b.iterations > a.iterations
    assert b.l1_errors[-1] <= 1e-10 < b.l1_errors[-2]


def test_build_csr_rejects_out_of_range(oracle):
    with pytest.raises(ValueError, match=r"edge #1 \(0,5\) has endpoint outside \[0,3\)"):
        oracle.build_csr(3, np.array([0, 0], np.uint64), np.array([1, 5], np.uint64))


def test_config_validation(oracle):
    g = oracle.build_csr(2, np.array([0, 1], np.uint64), np.array([1, 0], np.uint64))
    for kw in ({"damping": 0.0}, {"damping": 1.0}, {"threshold": 0.0}, {"max_iterations": 0}):
        with pytest.raises(ValueError):
            oracle.pagerank_ec(g, **kw)


@pytest.mark.slow
def test_config2_graph(oracle):
    rec = load("config2.json")
    n, s, d = oracle.random_sparse(rec["params"]["n"], rec["params"]["avg_degree"], rec["params"]["seed"])
    assert len(s) == rec["kept_draws"]
    g = oracle.build_csr(n, s, d)
    _graph_matches(g, rec["graph"])
    _run_matches(oracle.pagerank_ec(g, threshold=1e-10), rec["runs"]["ec_seq@1e-10"])


# ------------------------------------------------------------ edge-list ingest
def _check_parsed(p, c):
    assert p.error_line == c["error_line"], c["name"]
    assert p.error == c["error"], c["name"]
    if not c["error_line"]:
        assert p.n == c["n"], c["name"]
        assert p.edges.reshape(-1).tolist() == c["edges"], c["name"]


def test_oracle_parse_edge_list_golden(oracle):
    """fo_parse_edge_list == fpr::parse_edge_list on the reference's own test
    inputs (io_ingest_test.cpp:25-93), edge cases and seeded fuzz texts."""
    d = load("edge_list.json")
    assert len(d["cases"]) >= 150
    for c in d["cases"]:
        _check_parsed(oracle.parse_edge_list(c["text"].encode("latin-1")), c)


def test_oracle_parse_edge_list_large(oracle):
    from golden_util import sparse_text_from_edges

    big = load("edge_list.json")["large"]
    _, s, d = oracle.generate_rmat(12, 16, seed=7)
    text = sparse_text_from_edges(s, d)
    assert hashlib.sha256(text).hexdigest() == big["text_sha256"]
    p = oracle.parse_edge_list(text)
    assert (p.n, len(p.edges)) == (big["n"], big["m"])
    assert sha(p.edges.reshape(-1)) == big["edges_sha256"]


def test_fuzz_generator_is_deterministic():
    from golden_util import fuzz_text

    d = load("edge_list.json")
    fz = {c["name"]: c["text"] for c in d["cases"] if c["name"].startswith("fuzz_")}
    for s in (0, 1, 2, 57, 119):
        assert fuzz_text(s, 1 + s % 60, bad_rate=0.02 if s % 3 == 0 else 0.0).decode("latin-1") == fz[f"fuzz_{s}"]
