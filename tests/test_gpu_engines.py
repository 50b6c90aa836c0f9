"""GPU parity: B200 engines (through the C ABI) vs the oracle and the
reference-generated golden fixtures.

Tolerances (north_star): EC per iteration within 1e-12 relative (fp64);
fused within 1e-9 L1 of the reference fused result where that is well defined
(tight threshold), otherwise the geometric-tail bound against the
fixed point x*, with iteration counts reported beside it.
"""
import numpy as np
import pytest

import paper_2203_09284_b200 as fb
from golden_util import load, sha, small_edges, unhex
from oracle import Graph as OGraph

pytestmark = pytest.mark.gpu

EC_RTOL = 1e-12


def to_fb(g: OGraph) -> fb.Graph:
    return fb.Graph(g.n, g.m, g.in_start, g.in_src, g.out_degree)


def rel(a, b):
    return float(np.max(np.abs(a - b) / np.abs(b)))


@pytest.fixture(scope="module")
def config1(oracle):
    rec = load("config1.json")
    p = rec["params"]
    n, s, d = oracle.generate_rmat(p["scale"], p["edge_factor"], seed=p["seed"])
    g = oracle.build_csr(n, s, d)
    dg = fb.DeviceGraph.from_graph(to_fb(g))
    yield rec, g, dg
    dg.close()


def test_kats_all_engines(oracle):
    """SPEC.md:208-221 examples: 2-cycle, single dangling vertex, 3-vertex ..."""
    for name, rec in load("kat.json").items():
        g = oracle.build_csr(*small_edges(rec))
        cfg = fb.PageRankConfig(threshold=1e-15)
        ec = fb.pagerank_ec_b200(to_fb(g), cfg)
        assert ec.trace.iterations == rec["ec_seq"]["iterations"], name
        assert rel(ec.ranks.values, unhex(rec["ec_seq"]["ranks"])) <= EC_RTOL
        ref_err = unhex(rec["ec_seq"]["errors"])
        assert np.max(np.abs(ec.trace.errors - ref_err)) <= EC_RTOL * float(ec.ranks.values.max())
        one = fb.pagerank_ec_b200(to_fb(g), fb.PageRankConfig(threshold=1e-15, max_iterations=1))
        assert rel(one.ranks.values, unhex(rec["ec_one_step"])) <= EC_RTOL
        assert one.trace.iterations == 1
        with fb.DeviceGraph.from_graph(to_fb(g), wave_count=g.n) as dg:
            ls = dg.run(fb.ENGINE_FUSED_LOCKSTEP, cfg)
            ws = dg.wave_starts(g.n)
        if len(ws) == g.n + 1:  # one vertex per wave == fused_seq exactly
            assert ls.trace.iterations == rec["fused_seq"]["iterations"], name
            assert rel(ls.ranks.values, unhex(rec["fused_seq"]["ranks"])) <= EC_RTOL
        fu = fb.pagerank_fused_b200(to_fb(g), cfg)
        assert fu.trace.converged
        assert np.max(np.abs(fu.ranks.values - unhex(rec["dense"]))) <= 1e-12


def test_spec_literals():
    g = fb.Graph(2, 2, np.array([0, 1, 2], np.uint64), np.array([1, 0], np.uint64),
                 np.array([1, 1], np.uint64))
    r = fb.pagerank_ec_b200(g)
    assert r.trace.iterations == 1 and r.ranks.values.tolist() == [0.5, 0.5]
    g1 = fb.Graph(1, 0, np.array([0, 0], np.uint64), np.zeros(0, np.uint64), np.array([0], np.uint64))
    r = fb.pagerank_ec_b200(g1)
    assert r.trace.iterations == 2 and r.trace.converged
    assert r.ranks.values[0] == float.fromhex("0x1.3333333333334p-3")


def test_corpus_ec_and_oracle(oracle):
    """AC1 corpus: ec_b200 within 1e-12 relative of reference ec_seq with the
    same iteration count; fused engines agree with the dense oracle (AC1/AC2)."""
    for rec in load("corpus.json"):
        g = to_fb(oracle.build_csr(*small_edges(rec)))
        cfg = fb.PageRankConfig(threshold=1e-13)
        ec = fb.pagerank_ec_b200(g, cfg)
        assert ec.trace.iterations == rec["ec_seq"]["iterations"]
        assert rel(ec.ranks.values, unhex(rec["ec_seq"]["ranks"])) <= EC_RTOL
        dense = unhex(rec["dense"])
        for fn in (fb.pagerank_fused_b200, fb.pagerank_fused_lockstep_b200):
            r = fn(g, cfg)
            assert r.trace.converged
            assert np.max(np.abs(r.ranks.values - dense)) <= 1e-9  # SPEC AC2
            assert np.max(np.abs(r.ranks.values - unhex(rec["fused_seq"]["ranks"]))) <= 1e-9


def test_config1_ec_per_iteration(config1, oracle):
    """BASELINE: EC matches the reference per iteration within 1e-12 relative."""
    rec, g, dg = config1
    K = rec["runs"]["ec_seq@1e-10"]["iterations"]
    ref = oracle.pagerank_ec(g, threshold=1e-10, history_cap=K)
    for k in sorted({1, 2, 3, 5, 10, 20, 40, K - 1, K}):
        r = dg.run(fb.ENGINE_EC, fb.PageRankConfig(threshold=1e-10, max_iterations=k))
        assert r.trace.iterations == k
        assert rel(r.ranks.values, ref.history[k - 1]) <= EC_RTOL, k
    full = dg.run(fb.ENGINE_EC, fb.PageRankConfig(threshold=1e-10))
    assert full.trace.iterations == K == ref.iterations
    assert full.trace.converged
    # errors are differences of ranks: they agree to the rank tolerance, absolutely
    ref_err = unhex(rec["runs"]["ec_seq@1e-10"]["errors"])
    assert np.max(np.abs(full.trace.errors - ref_err)) <= EC_RTOL * float(ref.ranks.max())
    for i, h in rec["runs"]["ec_seq@1e-10"]["sample"].items():
        assert abs(full.ranks.values[int(i)] / float.fromhex(h) - 1) <= EC_RTOL
    # deterministic: a second run is bit-identical
    again = dg.run(fb.ENGINE_EC, fb.PageRankConfig(threshold=1e-10))
    np.testing.assert_array_equal(again.ranks.values, full.ranks.values)
    np.testing.assert_array_equal(again.trace.errors, full.trace.errors)


@pytest.mark.parametrize("waves", [0, 4, 16, 64])
def test_config1_lockstep_vs_restated_schedule(config1, oracle, waves):
    """Deterministic FusEd schedule restated on the CPU: per-sweep 1e-12 rel."""
    rec, g, dg = config1
    ws = dg.wave_starts(waves)
    assert ws[0] == 0 and ws[-1] == g.n and np.all(np.diff(ws.astype(np.int64)) > 0)
    ref = oracle.pagerank_lockstep(g, ws, threshold=1e-10, history_cap=200)
    with fb.DeviceGraph.from_graph(to_fb(g), wave_count=waves) as d2:
        for k in (1, 2, 5, ref.iterations):
            r = d2.run(fb.ENGINE_FUSED_LOCKSTEP, fb.PageRankConfig(threshold=1e-10, max_iterations=k))
            assert rel(r.ranks.values, ref.history[k - 1]) <= EC_RTOL
        r = d2.run(fb.ENGINE_FUSED_LOCKSTEP, fb.PageRankConfig(threshold=1e-10))
    assert r.trace.iterations == ref.iterations
    ec_iters = rec["runs"]["ec_seq@1e-10"]["iterations"]
    if len(ws) - 1 >= 8:
        assert r.trace.iterations < ec_iters  # Gauss-Seidel gain (F14)


def test_config1_fused_async(config1, oracle):
    """FusEd block-async: strict 1e-9 L1 vs reference fused_seq at 1e-13 (F8 ii);
    at 1e-10 the geometric-tail bound vs x* (F8 iii); iterations reported."""
    rec, g, dg = config1
    tight = dg.run(fb.ENGINE_FUSED, fb.PageRankConfig(threshold=1e-13))
    ref_tight = oracle.pagerank_fused_seq(g, threshold=1e-13)
    assert sha(ref_tight.ranks) == rec["runs"]["fused_seq@1e-13"]["ranks_sha256"]
    l1 = fb.l1_norm(tight.ranks.values, ref_tight.ranks)
    assert l1 <= 1e-9, l1
    xstar = oracle.pagerank_ec(g, threshold=1e-16, max_iterations=400).ranks
    r = dg.run(fb.ENGINE_FUSED, fb.PageRankConfig(threshold=1e-10))
    bound = g.n * 1e-10 * 0.85 / 0.15
    assert r.trace.converged
    assert fb.l1_norm(r.ranks.values, xstar) <= bound
    print(f"\nconfig1 fused_b200 iterations={r.trace.iterations} "
          f"(fused_seq {rec['runs']['fused_seq@1e-10']['iterations']}, "
          f"ec_seq {rec['runs']['ec_seq@1e-10']['iterations']}) "
          f"L1 vs x*={fb.l1_norm(r.ranks.values, xstar):.3e}")


def test_l1_norm_stop_rule(config1, oracle):
    rec, g, dg = config1
    ref = oracle.pagerank_ec(g, threshold=1e-10, norm=1)
    with fb.DeviceGraph.from_graph(to_fb(g), norm=fb.NORM_L1) as d2:
        r = d2.run(fb.ENGINE_EC, fb.PageRankConfig(threshold=1e-10))
    assert r.trace.iterations == ref.iterations
    assert np.max(np.abs(r.trace.l1_errors - ref.l1_errors)) <= EC_RTOL * float(ref.ranks.sum())


def test_validation_messages():
    g = fb.Graph(2, 2, np.array([0, 1, 2], np.uint64), np.array([1, 0], np.uint64),
                 np.array([1, 1], np.uint64))
    cases = [({"damping": 0.0}, "damping must be in"), ({"damping": 1.0}, "damping must be in"),
             ({"threshold": 0.0}, "threshold must be positive"),
             ({"max_iterations": 0}, "max_iterations must be positive"),
             ({"thread_count": 0}, "thread_count must be positive")]
    for kw, msg in cases:
        with pytest.raises(ValueError, match=msg):
            fb.pagerank_ec_b200(g, fb.PageRankConfig(**kw))
    bad = fb.Graph(2, 2, np.array([0, 1, 2], np.uint64), np.array([1, 7], np.uint64),
                   np.array([1, 1], np.uint64))
    with pytest.raises(ValueError, match="outside"):
        fb.pagerank_ec_b200(bad)
    empty = fb.Graph(0, 0, np.array([0], np.uint64), np.zeros(0, np.uint64), np.zeros(0, np.uint64))
    with pytest.raises(ValueError, match="pagerank: graph has no vertices"):
        fb.pagerank_ec_b200(empty)


def test_max_iterations_nonconvergence(config1):
    rec, g, dg = config1
    r = dg.run(fb.ENGINE_EC, fb.PageRankConfig(threshold=1e-15, max_iterations=3))
    assert r.trace.iterations == 3 and not r.trace.converged
    assert r.ranks.final_error == r.trace.errors[-1]


def test_upload_download_roundtrip(config1):
    rec, g, dg = config1
    back = dg.download()
    assert back.m == g.m
    np.testing.assert_array_equal(back.in_start, g.in_start)
    np.testing.assert_array_equal(back.in_src, g.in_src)
    np.testing.assert_array_equal(back.out_degree, g.out_degree)


@pytest.mark.parametrize("reorder,pb", [(True, None), ("sources", None), ("blocks", None), ("blocks", True),
                                        (True, True)])
def test_reorder_option_preserves_results(config1, oracle, reorder, pb, monkeypatch):
    """FPR_B200_OPT_REORDER renumbers vertices internally by out-degree,
    FPR_B200_OPT_REORDER_SOURCES puts the vertices with out-edges first,
    FPR_B200_OPT_REORDER_BLOCKS orders by degree inside each source-chunk
    block (small chunks here, so that the blocks matter); EC
    results come back in the caller's ids, per-iteration within 1e-12, with
    the same iteration count (Jacobi is relabel-invariant)."""
    rec, g, dg = config1
    monkeypatch.setenv("FPR_B200_PB_CHUNK_SHIFT", "12")
    ref = oracle.pagerank_ec(g, threshold=1e-10, history_cap=3)
    with fb.DeviceGraph.from_graph(to_fb(g), reorder=reorder, pb=pb) as d2:
        r1 = d2.run(fb.ENGINE_EC, fb.PageRankConfig(threshold=1e-10, max_iterations=3))
        assert rel(r1.ranks.values, ref.history[2]) <= EC_RTOL
        r = d2.run(fb.ENGINE_EC, fb.PageRankConfig(threshold=1e-10))
        fu = d2.run(fb.ENGINE_FUSED, fb.PageRankConfig(threshold=1e-10))
        with pytest.raises(ValueError, match="REORDER"):
            d2.download()
    assert r.trace.iterations == ref.iterations
    assert rel(r.ranks.values, ref.ranks) <= EC_RTOL
    xstar = oracle.pagerank_ec(g, threshold=1e-16, max_iterations=400).ranks
    assert fu.trace.converged and fb.l1_norm(fu.ranks.values, xstar) <= g.n * 1e-10 * 0.85 / 0.15


@pytest.mark.parametrize("share", ["0", "0.5", "1"])
def test_pinned_upload_split(config1, share, monkeypatch):
    """Pinned sources: the first (1-share) of in_src is DMA'd raw and narrowed
    on the device, the rest narrowed by host threads (AVX-512) into the
    pinned ring -- both halves land bit-exactly and both range-check."""
    import torch

    rec, g, dg = config1
    monkeypatch.setenv("FPR_B200_HOST_NARROW", share)

    def pinned(a):
        t = torch.empty(len(a), dtype=torch.int64, pin_memory=True)
        v = t.numpy().view(np.uint64)
        v[:] = a
        return t, v

    keep = [pinned(g.in_start), pinned(g.in_src), pinned(g.out_degree)]
    pg = fb.Graph(g.n, g.m, keep[0][1], keep[1][1], keep[2][1])
    with fb.DeviceGraph.from_graph(pg) as d2:
        back = d2.download()
    np.testing.assert_array_equal(back.in_src, g.in_src)
    np.testing.assert_array_equal(back.out_degree, g.out_degree)
    for pos in (0, g.m // 2 + 17, g.m - 1):  # raw half, either side of the split, host half
        src = keep[1][1]
        old = int(src[pos])
        src[pos] = g.n + pos
        try:
            with pytest.raises(ValueError, match="outside"):
                fb.DeviceGraph.from_graph(pg)
        finally:
            src[pos] = old


@pytest.mark.parametrize("shift,chunk_shift,reorder,piece,lpiece",
                         [(13, 20, False, 0, 0), (5, 4, False, 0, 0), (9, 12, False, 0, 0), (12, 10, True, 0, 0),
                          (7, 6, False, 0, 0), (13, 20, False, 1000, 0), (9, 12, True, 77, 0),
                          (13, 20, False, 0, 1000), (9, 12, False, 77, 333), (13, 16, False, 0, 1)])
def test_pb_ec_matches_oracle(config1, oracle, shift, chunk_shift, reorder, piece, lpiece, monkeypatch):
    """FPR_B200_OPT_PB: propagation-blocked EC sweeps (gather pass summing
    each row's run into the bin-major partial-sum stream + shared-memory bin
    accumulation) give the reference's per-iteration ranks within 1e-12
    relative and its iteration count, from one bin/chunk to thousands of
    each, with whole bins and with bins split into units finished by their
    last-arriving CTA, and with the layout built from bins cut into pieces
    of `lpiece` edges (pieces start mid-row; down to one edge per piece)."""
    rec, g, dg = config1
    monkeypatch.setenv("FPR_B200_PB_SHIFT", str(shift))
    monkeypatch.setenv("FPR_B200_PB_CHUNK_SHIFT", str(chunk_shift))
    if piece:  # heavy bins split into phase-2 units of about `piece` entries
        monkeypatch.setenv("FPR_B200_PB_PIECE", str(piece))
    if lpiece:  # the layout's pieces (default 2^18 edges: only hub bins split)
        monkeypatch.setenv("FPR_B200_PB_LAYOUT_PIECE", str(lpiece))
    ref = oracle.pagerank_ec(g, threshold=1e-10, history_cap=3)
    with fb.DeviceGraph.from_graph(to_fb(g), pb=True, reorder=reorder) as d2:
        r1 = d2.run(fb.ENGINE_EC, fb.PageRankConfig(threshold=1e-10, max_iterations=1))
        assert rel(r1.ranks.values, ref.history[0]) <= EC_RTOL
        r3 = d2.run(fb.ENGINE_EC, fb.PageRankConfig(threshold=1e-10, max_iterations=3))
        assert rel(r3.ranks.values, ref.history[2]) <= EC_RTOL
        r = d2.run(fb.ENGINE_EC, fb.PageRankConfig(threshold=1e-10))
        r2 = d2.run(fb.ENGINE_EC, fb.PageRankConfig(threshold=1e-10))
        fu = d2.run(fb.ENGINE_FUSED, fb.PageRankConfig(threshold=1e-10))  # FUSED: lockstep on PB sweeps
    assert r.sweep == fb.SWEEP_PB and fu.sweep == fb.SWEEP_PB
    assert r.trace.iterations == ref.iterations and r.trace.converged
    assert rel(r.ranks.values, ref.ranks) <= EC_RTOL
    assert np.max(np.abs(r.trace.errors - ref.errors)) <= EC_RTOL * float(ref.ranks.max())
    # fixed-point row sums: a second run gives the same bits
    assert np.array_equal(r.ranks.values.view(np.uint64), r2.ranks.values.view(np.uint64))
    assert np.array_equal(r.trace.errors, r2.trace.errors) and np.array_equal(r.trace.l1_errors, r2.trace.l1_errors)
    assert fu.trace.converged


@pytest.mark.parametrize("shift,chunk_shift,waves,piece", [(13, 20, 0, 0), (9, 12, 4, 0), (7, 10, 16, 300),
                                                         (5, 6, 64, 0), (9, 12, 3, 77), (13, 20, 100, 0)])
def test_pb_lockstep_vs_restated_schedule(config1, oracle, shift, chunk_shift, waves, piece, monkeypatch):
    """FPR_B200_OPT_PB + the lockstep engine: S waves of consecutive bins,
    each gathered from and written back to the one contribution vector, is
    the deterministic FusEd schedule of fo_pagerank_lockstep at bin-aligned
    wave starts: per-sweep 1e-12 relative and the same sweep count (more
    waves than bins included: the waves shrink to one bin each)."""
    rec, g, dg = config1
    monkeypatch.setenv("FPR_B200_PB_SHIFT", str(shift))
    monkeypatch.setenv("FPR_B200_PB_CHUNK_SHIFT", str(chunk_shift))
    if piece:
        monkeypatch.setenv("FPR_B200_PB_PIECE", str(piece))
    with fb.DeviceGraph.from_graph(to_fb(g), pb=True, wave_count=waves) as d2:
        ws = d2.wave_starts(waves)
        assert ws[0] == 0 and ws[-1] == g.n and np.all(np.diff(ws.astype(np.int64)) > 0)
        assert np.all(ws[:-1] % (1 << shift) == 0)
        ref = oracle.pagerank_lockstep(g, ws, threshold=1e-10, history_cap=200)
        for k in (1, 2, 5, ref.iterations):
            r = d2.run(fb.ENGINE_FUSED_LOCKSTEP, fb.PageRankConfig(threshold=1e-10, max_iterations=k))
            assert rel(r.ranks.values, ref.history[k - 1]) <= EC_RTOL
        r = d2.run(fb.ENGINE_FUSED_LOCKSTEP, fb.PageRankConfig(threshold=1e-10))
        ec = d2.run(fb.ENGINE_EC, fb.PageRankConfig(threshold=1e-10))  # both plans cached side by side
    assert r.trace.iterations == ref.iterations and r.trace.converged
    assert rel(r.ranks.values, ref.ranks) <= EC_RTOL
    assert ec.trace.iterations == rec["runs"]["ec_seq@1e-10"]["iterations"]
    if len(ws) - 1 >= 8:
        assert r.trace.iterations < ec.trace.iterations  # Gauss-Seidel gain


def test_pb_l1_rule_matches_pull(config1):
    """The L1 stop rule stops the propagation-blocked engine at the pull
    engine's iteration with the same trace (within the 1e-12 tolerance)."""
    rec, g, dg = config1
    cfg = fb.PageRankConfig(threshold=1e-9)
    with fb.DeviceGraph.from_graph(to_fb(g), norm=fb.NORM_L1) as a, \
            fb.DeviceGraph.from_graph(to_fb(g), norm=fb.NORM_L1, pb=True) as b:
        ra, rb = a.run(fb.ENGINE_EC, cfg), b.run(fb.ENGINE_EC, cfg)
    assert ra.trace.iterations == rb.trace.iterations
    assert rel(rb.ranks.values, ra.ranks.values) <= EC_RTOL
    assert np.max(np.abs(ra.trace.l1_errors - rb.trace.l1_errors)) <= 1e-12


def test_sweep_kind_auto_and_forced(config1, oracle, monkeypatch):
    """Default options let the library pick the sweep: pull while the
    contribution vector fits L2 (config 1), propagation-blocked past the size
    rule (lowered here through FPR_B200_PB_AUTO_BYTES); pb=False forces the
    pull sweep.  Every choice keeps the reference's per-iteration parity."""
    rec, g, dg = config1
    ref = oracle.pagerank_ec(g, threshold=1e-10)
    cfg = fb.PageRankConfig(threshold=1e-10)
    with fb.DeviceGraph.from_graph(to_fb(g)) as d:
        r = d.run(fb.ENGINE_EC, cfg)
    assert r.sweep == fb.SWEEP_PULL
    monkeypatch.setenv("FPR_B200_PB_AUTO_BYTES", "1024")
    with fb.DeviceGraph.from_graph(to_fb(g)) as d, fb.DeviceGraph.from_graph(to_fb(g), pb=False) as dp:
        before = d.layout_info()
        ra, rp = d.run(fb.ENGINE_EC, cfg), dp.run(fb.ENGINE_EC, cfg)
        fa = d.run(fb.ENGINE_FUSED, cfg)
        after, pull = d.layout_info(), dp.layout_info()
    assert ra.sweep == fb.SWEEP_PB and fa.sweep == fb.SWEEP_PB and rp.sweep == fb.SWEEP_PULL
    # fpr_b200_graph_layout_info: the PB layout exists after the first PB run;
    # one partial sum per run: at most one per entry (+ up to 7 pad places per bin)
    assert before["sweep"] == fb.SWEEP_PB and before["runs"] == 0
    assert after["runs"] > 0 and after["pieces"] > 0 and after["tiles"] > 0
    assert after["runs"] <= g.m + 8 * (g.n // 8192 + 1)
    assert pull["sweep"] == fb.SWEEP_PULL and pull["runs"] == 0
    for x in (ra, rp):
        assert x.trace.iterations == ref.iterations
        assert rel(x.ranks.values, ref.ranks) <= EC_RTOL
    assert fa.trace.converged


def test_pb_rejects_bad_geometry(config1, monkeypatch):
    """Bins wider than the uint16 row offset (or too narrow) are an argument
    error at the first EC run, not a silent fallback."""
    rec, g, dg = config1
    monkeypatch.setenv("FPR_B200_PB_SHIFT", "17")
    with fb.DeviceGraph.from_graph(to_fb(g), pb=True) as d2:
        with pytest.raises(ValueError, match="propagation-blocked"):
            d2.run(fb.ENGINE_EC, fb.PageRankConfig(threshold=1e-10))


def test_pb_random_geometries(oracle, monkeypatch):
    """Randomised propagation-blocked layouts against the oracle: R-MAT and
    uniform graphs of random size and degree, random bin / chunk shifts,
    layout pieces, accumulate units and wave counts (hot copy on and off:
    chunks below 32 sources have none).  EC: the reference's iteration count
    and ranks within 1e-12; lockstep: converged; reruns bit-equal."""
    import os

    rng = np.random.default_rng(int(os.environ.get("FPR_TEST_SEED", "2026")))
    for case in range(int(os.environ.get("FPR_TEST_CASES", "16"))):
        if case % 2:
            n, s, d = oracle.generate_rmat(int(rng.integers(5, 15)), int(rng.integers(1, 24)),
                                           seed=int(rng.integers(1 << 30)))
        else:
            n0 = int(rng.integers(1, 40000))
            n, s, d = oracle.random_sparse(n0, int(rng.integers(1, 20)), int(rng.integers(1 << 30)))
        g = oracle.build_csr(n, s, d)
        if g.n == 0:
            continue
        env = {"FPR_B200_PB_SHIFT": str(int(rng.integers(5, 14))),
               "FPR_B200_PB_CHUNK_SHIFT": str(int(rng.integers(3, 16))),
               "FPR_B200_PB_LAYOUT_PIECE": str(int(rng.choice([1, 17, 500, 1 << 18]))),
               "FPR_B200_PB_PIECE": str(int(rng.choice([32, 300, 1 << 16])))}
        for k, v in env.items():
            monkeypatch.setenv(k, v)
        ref = oracle.pagerank_ec(g, threshold=1e-10)
        with fb.DeviceGraph.from_graph(to_fb(g), pb=True, wave_count=int(rng.integers(0, 9))) as dg:
            r = dg.run(fb.ENGINE_EC, fb.PageRankConfig(threshold=1e-10))
            r2 = dg.run(fb.ENGINE_EC, fb.PageRankConfig(threshold=1e-10))
            lk = dg.run(fb.ENGINE_FUSED_LOCKSTEP, fb.PageRankConfig(threshold=1e-10))
        assert r.sweep == fb.SWEEP_PB, (case, env)
        assert r.trace.iterations == ref.iterations, (case, env)
        assert rel(r.ranks.values, ref.ranks) <= EC_RTOL, (case, env)
        assert np.array_equal(r.ranks.values.view(np.uint64), r2.ranks.values.view(np.uint64)), (case, env)
        assert lk.trace.converged, (case, env)
