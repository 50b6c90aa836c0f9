"""The multi-device C ABI (fpr_b200_mgpu_*, fpr_b200_options.devices) on ONE
B200: P parts of the same graph, all on device 0, driven from this thread.
Parts sharing a device run their sweeps one after the other on their own
streams and exchange contributions through the sweep epilogue's stores into
every part's vector -- the code path that stores across NVLink when the
devices differ.  EC must equal the oracle per 1e-12 relative with the same
iteration count; FusEd converges within the tail bound."""
import ctypes as C

import numpy as np
import pytest

import paper_2203_09284_b200 as fb

pytestmark = pytest.mark.gpu
T = 1e-10


@pytest.fixture(scope="module")
def rmat16(oracle):
    n, s, d = oracle.generate_rmat(16, 16, seed=1)
    g = oracle.build_csr(n, s, d)
    return g, fb.Graph(g.n, g.m, g.in_start, g.in_src, g.out_degree)


@pytest.mark.parametrize("P,pb", [(1, False), (2, False), (3, False), (5, False), (8, False), (2, True), (3, True),
                                  (8, True)])
def test_mgpu_ec_matches_oracle(oracle, rmat16, P, pb, monkeypatch):
    """pb=True: propagation-blocked part sweeps (bins over the part's rows,
    chunks over the exchange space, the finalize storing into the peers),
    small chunks so that every part walks several."""
    g, hg = rmat16
    monkeypatch.setenv("FPR_B200_PB_CHUNK_SHIFT", "12")
    ref = oracle.pagerank_ec(g, threshold=T, history_cap=2)
    with fb.MultiDeviceGraph.from_graph(hg, [0] * P, pb=pb) as mg:
        assert mg.nparts == P and mg.bounds[0] == 0 and mg.bounds[-1] == g.n
        r = mg.run(fb.ENGINE_EC, fb.PageRankConfig(threshold=T))
        r2 = mg.run(fb.ENGINE_EC, fb.PageRankConfig(threshold=T, max_iterations=2))
        fu = mg.run(fb.ENGINE_FUSED, fb.PageRankConfig(threshold=T))
    assert r.sweep == (fb.SWEEP_PB if pb else fb.SWEEP_PULL)
    assert r.trace.iterations == ref.iterations and r.trace.converged
    assert float(np.max(np.abs(r.ranks.values - ref.ranks) / ref.ranks)) <= 1e-12
    assert np.max(np.abs(r.trace.errors - ref.errors)) <= 1e-12 * float(ref.ranks.max())
    assert float(np.max(np.abs(r2.ranks.values - ref.history[1]) / ref.history[1])) <= 1e-12
    xstar = oracle.pagerank_ec(g, threshold=1e-16, max_iterations=400).ranks
    assert fu.trace.converged and oracle.l1_norm(fu.ranks.values, xstar) <= g.n * T * 0.85 / 0.15


@pytest.mark.parametrize("batch", ["1", "3", "64"])
def test_mgpu_device_stop_batches(rmat16, batch, monkeypatch):
    """The driver enqueues `batch` iterations between reads of the device-side
    gate; sweeps issued past the stopping iteration are no-ops.  Any batch
    gives the same iteration count, trace and rank bits."""
    g, hg = rmat16
    cfg = fb.PageRankConfig(threshold=T)
    with fb.MultiDeviceGraph.from_graph(hg, [0, 0, 0]) as mg:
        base = mg.run(fb.ENGINE_EC, cfg)
        monkeypatch.setenv("FPR_B200_MGPU_BATCH", batch)
        r = mg.run(fb.ENGINE_EC, cfg)
        cap = mg.run(fb.ENGINE_EC, fb.PageRankConfig(threshold=T, max_iterations=5))
    assert r.trace.iterations == base.trace.iterations
    assert np.array_equal(r.trace.errors, base.trace.errors)
    assert np.array_equal(r.ranks.values, base.ranks.values)
    assert cap.trace.iterations == 5 and not cap.trace.converged


def test_mgpu_generate_equals_host_view(rmat16):
    """Every device generating the graph itself gives the same parts, the
    same iterations and the same bits as the parts uploaded from the host."""
    g, hg = rmat16
    cfg = fb.PageRankConfig(threshold=T)
    with fb.MultiDeviceGraph.generate_rmat(fb.RmatParams(16, 16, seed=1), [0, 0, 0]) as a, \
            fb.MultiDeviceGraph.from_graph(hg, [0, 0, 0]) as b:
        assert (a.n, a.m) == (b.n, b.m) and np.array_equal(a.bounds, b.bounds)
        ra, rb = a.run(fb.ENGINE_EC, cfg), b.run(fb.ENGINE_EC, cfg)
    assert ra.trace.iterations == rb.trace.iterations
    assert np.array_equal(ra.ranks.values, rb.ranks.values)


def test_pagerank_one_shot_with_device_list(oracle, rmat16):
    """fpr_b200_pagerank() with opts.ndevices > 1 takes the multi-device path
    (the call the C++ drop-in makes with a device list in its options)."""
    g, hg = rmat16
    ref = oracle.pagerank_ec(g, threshold=T)
    ins, src, od = (np.ascontiguousarray(a, dtype=np.uint64) for a in (g.in_start, g.in_src, g.out_degree))
    view = fb._GraphView(g.n, g.m, ins.ctypes.data, src.ctypes.data, od.ctypes.data)
    devs = (C.c_int32 * 4)(0, 0, 0, 0)
    opts = fb._options()
    opts.devices = C.cast(devs, C.POINTER(C.c_int32))
    opts.ndevices = 4
    ranks = np.empty(g.n)
    errs = np.empty(1000)
    res = fb._Result()
    cfg = fb.PageRankConfig(threshold=T)._c()
    fb._check(fb.lib().fpr_b200_pagerank(C.byref(view), fb.ENGINE_EC, C.byref(cfg), C.byref(opts),
                                         ranks.ctypes.data, errs.ctypes.data, 1000, C.byref(res)))
    assert res.iterations == ref.iterations and res.converged
    assert float(np.max(np.abs(ranks - ref.ranks) / ref.ranks)) <= 1e-12


def test_mgpu_argument_errors(rmat16):
    g, hg = rmat16
    with pytest.raises(ValueError, match="out of range"):
        fb.MultiDeviceGraph.from_graph(hg, [0, 999])
    with fb.MultiDeviceGraph.from_graph(hg, [0, 0]) as mg:
        with pytest.raises(ValueError, match="EC and FUSED"):
            mg.run(fb.ENGINE_FUSED_LOCKSTEP, fb.PageRankConfig(threshold=T))
        with pytest.raises(ValueError, match="damping"):
            mg.run(fb.ENGINE_EC, fb.PageRankConfig(damping=1.5))


@pytest.mark.parametrize("config,P", [("4", 2), ("4", 3), ("4", 8), ("5", 2), ("5", 4), ("5", 8)])
def test_mgpu_full_size_equals_single_gpu(config, P):
    """Configs 4/5 split into P destination-range parts on this one GPU, each
    part generating the graph on its device and running propagation-blocked
    part sweeps (the library's choice there), equal the single-GPU EC: the
    same iteration count and ranks within 1e-12 (the per-part
    sums are the same fixed regroupings as on one GPU, up to the part split)."""
    cfg = fb.PageRankConfig(threshold=T)
    if config == "4":
        gp = fb._GenParams(fb.GEN_CHUNGLU, 0, 0, 0.0, 0.0, 0.0, 0.0, 1 << 26, 0, 4, 1_200_000_000, 2.1, 1_000_000)
        one = fb.DeviceGraph.generate_chunglu(1 << 26, 1_200_000_000, seed=4)
    else:
        p = fb.RmatParams(28, 16, seed=5)
        gp = fb._GenParams(fb.GEN_RMAT, p.scale, p.edge_factor, p.a, p.b, p.c, p.d, 0, 0, p.seed)
        one = fb.DeviceGraph.generate_rmat(p)
    with one:
        ref = one.run(fb.ENGINE_EC, cfg)
    keep = []
    h = C.c_void_p()
    fb._check(fb.lib().fpr_b200_mgpu_generate(C.byref(gp), C.byref(fb.MultiDeviceGraph._opts([0] * P, fb.NORM_LINF,
                                                                                            keep)), C.byref(h)))
    with fb.MultiDeviceGraph(h.value, [0] * P) as mg:
        r = mg.run(fb.ENGINE_EC, cfg)
    assert r.sweep == fb.SWEEP_PB
    assert r.trace.iterations == ref.trace.iterations
    assert float(np.max(np.abs(r.ranks.values - ref.ranks.values) / ref.ranks.values)) <= 1e-12
    print(f"\nconfig{config} x{P} parts: {r.trace.iterations} iterations, {r.solve_ms:.0f} ms "
          f"(one GPU, parts in turn; single-part {ref.solve_ms:.0f} ms)")


def test_mgpu_random_parts(oracle, monkeypatch):
    """Randomised multi-part solves on one GPU: random graphs, 2-6 parts,
    pull or propagation-blocked parts with random geometries, random batch
    sizes of the device-side stop.  EC equals the oracle (iterations, 1e-12)."""
    import os

    rng = np.random.default_rng(int(os.environ.get("FPR_TEST_SEED", "7")))
    for case in range(int(os.environ.get("FPR_TEST_CASES", "8"))):
        if case % 2:
            n, s, d = oracle.generate_rmat(int(rng.integers(6, 14)), int(rng.integers(2, 20)),
                                           seed=int(rng.integers(1 << 30)))
        else:
            n, s, d = oracle.random_sparse(int(rng.integers(50, 30000)), int(rng.integers(1, 16)),
                                           int(rng.integers(1 << 30)))
        g = oracle.build_csr(n, s, d)
        P = int(rng.integers(2, 7))
        pb = bool(rng.integers(0, 2))
        monkeypatch.setenv("FPR_B200_PB_SHIFT", str(int(rng.integers(5, 14))))
        monkeypatch.setenv("FPR_B200_PB_CHUNK_SHIFT", str(int(rng.integers(4, 16))))
        monkeypatch.setenv("FPR_B200_MGPU_BATCH", str(int(rng.integers(1, 12))))
        ref = oracle.pagerank_ec(g, threshold=T)
        hg = fb.Graph(g.n, g.m, g.in_start, g.in_src, g.out_degree)
        with fb.MultiDeviceGraph.from_graph(hg, [0] * P, pb=pb) as mg:
            r = mg.run(fb.ENGINE_EC, fb.PageRankConfig(threshold=T))
        assert r.trace.iterations == ref.iterations, (case, P, pb)
        assert float(np.max(np.abs(r.ranks.values - ref.ranks) / ref.ranks)) <= 1e-12, (case, P, pb)
