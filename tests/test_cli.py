"""SPEC bench-cli contract for the B200 engines."""
import csv
import io

import numpy as np
import pytest

from paper_2203_09284_b200 import Graph
from paper_2203_09284_b200.cache import save_cache
from paper_2203_09284_b200.cli import CSV_COLUMNS, EXIT_IO, EXIT_NONCONV, EXIT_OK, EXIT_USAGE, main


def _run(argv):
    out = io.StringIO()
    rc = main(argv, out)
    return rc, out.getvalue()


def test_usage_errors():
    assert _run(["run"])[0] == EXIT_USAGE  # no graph source
    assert _run(["run", "--rmat", "bad"])[0] == EXIT_USAGE
    assert _run(["nosuch"])[0] == EXIT_USAGE
    assert _run(["run", "--rmat", "4:2:1", "--engine", "ec_seq"])[0] == EXIT_USAGE


def test_option_usage_errors():
    assert _run(["gen", "--rmat", "4:2:1", "--out", "/dev/null", "--reorder", "degree"])[0] == EXIT_USAGE
    assert _run(["run", "--rmat", "4:2:1", "--reorder", "bfs"])[0] == EXIT_USAGE


def test_missing_file_is_io_error(tmp_path):
    assert _run(["run", "--graph", str(tmp_path / "missing.fprg")])[0] == EXIT_IO


@pytest.mark.gpu
def test_run_two_cycle(tmp_path):
    p = str(tmp_path / "c2.fprg")
    save_cache(Graph(2, 2, np.array([0, 1, 2], np.uint64), np.array([1, 0], np.uint64),
                     np.array([1, 1], np.uint64)), p)
    rc, text = _run(["run", "--graph", p, "--engine", "ec_b200"])
    assert rc == EXIT_OK
    assert "iterations=1" in text and text.splitlines()[1] == "0:0.5, 1:0.5"
    rc, _ = _run(["run", "--rmat", "10:16:1", "--threshold", "1e-15", "--max-iters", "3"])
    assert rc == EXIT_NONCONV


@pytest.mark.gpu
def test_bench_csv_schema(tmp_path):
    out = tmp_path / "b.csv"
    rc, _ = _run(["bench", "--rmat", "8:16:1", "--engines", "ec_b200,fused_lockstep_b200",
                  "--thresholds", "1e-8,1e-12", "--out", str(out)])
    assert rc == EXIT_OK
    rows = list(csv.DictReader(open(out)))
    assert list(rows[0].keys()) == CSV_COLUMNS and len(rows) == 4
    for r in rows:
        if r["engine"] == "ec_b200":
            assert float(r["l1_vs_seq_ec"]) == 0.0
        assert r["converged"] == "true"


@pytest.mark.gpu
def test_bench_library_options(tmp_path):
    """--pb / --reorder / --waves reach the library: the propagation-blocked
    EC and lockstep engines on a sources-first renumbered graph converge, and
    PB EC matches the plain EC row's iteration count."""
    out = tmp_path / "o.csv"
    rc, _ = _run(["bench", "--rmat", "10:16:1", "--engines", "ec_b200,fused_lockstep_b200", "--thresholds", "1e-10",
                  "--pb", "--reorder", "sources", "--waves", "4", "--out", str(out)])
    assert rc == EXIT_OK
    rows = {r["engine"]: r for r in csv.DictReader(open(out))}
    assert all(r["converged"] == "true" for r in rows.values())
    plain = tmp_path / "p.csv"
    assert _run(["bench", "--rmat", "10:16:1", "--engines", "ec_b200", "--thresholds", "1e-10",
                 "--out", str(plain)])[0] == EXIT_OK
    assert next(csv.DictReader(open(plain)))["iterations"] == rows["ec_b200"]["iterations"]


@pytest.mark.gpu
def test_gen_and_compare(tmp_path):
    p = str(tmp_path / "g.fprg")
    assert _run(["gen", "--rmat", "6:4:3", "--format", "fprg", "--out", p])[0] == EXIT_OK
    rc, text = _run(["compare", "--graph", p, "--threshold", "1e-12"])
    assert rc == EXIT_OK and text.startswith("iteration,ec_b200,fused_b200,fused_lockstep_b200")


@pytest.mark.gpu
def test_gen_writes_the_generated_edgeset(tmp_path):
    """SPEC cmd_gen: scale=3, edge_factor=2, seed=1 -> exactly 16 edge lines
    (the raw draws: self-loops and duplicates kept), header comments with the
    parameters and seed, byte-identical on a rerun, and re-ingested by run."""
    a, b = tmp_path / "a.txt", tmp_path / "b.txt"
    assert _run(["gen", "--rmat", "3:2:1", "--out", str(a)])[0] == EXIT_OK
    assert _run(["gen", "--rmat", "3:2:1", "--out", str(b)])[0] == EXIT_OK
    text = a.read_bytes()
    assert text == b.read_bytes()
    lines = text.decode().splitlines()
    edges = [l for l in lines if l and not l.startswith("#")]
    assert len(edges) == 16 and any("seed=1" in l for l in lines if l.startswith("#"))
    rc, out = _run(["run", "--edges", str(a), "--threshold", "1e-10"])
    assert rc == EXIT_OK and "converged=true" in out


@pytest.mark.gpu
def test_generate_edges_are_the_reference_draws(oracle):
    """fb.generate_edges draws on the device exactly the EdgeSet of the
    reference's generate_rmat (pinned by tests/golden/rmat_s10_seed42.json's
    draw digests) and random_sparse's kept draws (the oracle restatement)."""
    import paper_2203_09284_b200 as fb
    from golden_util import load, sha

    rec = load("rmat_s10_seed42.json")
    es = fb.generate_edges("rmat", params=fb.RmatParams(10, 16, seed=42))
    assert sha(es.edges[:, 0].copy()) == rec["draws_sha256"]["src"]
    assert sha(es.edges[:, 1].copy()) == rec["draws_sha256"]["dst"]
    n, s, d = oracle.random_sparse(1000, 8, 5)
    eu = fb.generate_edges("uniform", n=1000, avg_degree=8, seed=5)
    assert np.array_equal(eu.edges[:, 0], s) and np.array_equal(eu.edges[:, 1], d)


@pytest.mark.gpu
def test_bench_thread_list_and_failed_cells(tmp_path):
    """SPEC cmd_bench: the cross-product over a --threads list, and a cell
    that fails (threshold 0 is invalid) is a converged=false row, not an
    aborted sweep."""
    out = tmp_path / "t.csv"
    rc, _ = _run(["bench", "--rmat", "8:16:1", "--engines", "ec_b200,fused_b200", "--thresholds", "1e-8,0",
                  "--threads", "1,4", "--out", str(out)])
    assert rc == EXIT_OK
    rows = list(csv.DictReader(open(out)))
    assert len(rows) == 2 * 2 * 2
    assert sorted({r["threads"] for r in rows}) == ["1", "4"]
    for r in rows:
        assert r["converged"] == ("true" if r["threshold"] == "1e-08" else "false")
