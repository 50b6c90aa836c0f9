"""BASELINE configs 3-5 at full size on the device: generation (K5/K4 + the
config-3 relabel), build_csr invariants checked on the device, and
size-independent PageRank properties the oracle cannot reach in test time:
  * relabel invariance of the EC iteration count (config 3 vs natural order);
  * fixed-point residual: one more Jacobi step moves no rank by more than
    10*threshold/(1-d);
  * lower bound: every rank >= (1-d)/n - 1e-12;
  * EC and FusEd agree within the geometric-tail bound n*delta*d/(1-d).
"""
import numpy as np
import pytest

import paper_2203_09284_b200 as fb

pytestmark = pytest.mark.gpu
D = 0.85
T = 1e-10


def _properties(dg, name):
    cfg = fb.PageRankConfig(threshold=T)
    ec = dg.run(fb.ENGINE_EC, cfg)
    assert ec.trace.converged
    k = ec.trace.iterations
    nxt = dg.run(fb.ENGINE_EC, fb.PageRankConfig(threshold=T, max_iterations=k + 1))
    assert float(np.max(np.abs(nxt.ranks.values - ec.ranks.values))) <= 10 * T / (1 - D)
    assert float(ec.ranks.values.min()) >= (1 - D) / dg.n - 1e-12
    fu = dg.run(fb.ENGINE_FUSED, cfg)
    assert fu.trace.converged
    assert fb.l1_norm(fu.ranks.values, ec.ranks.values) <= 2 * dg.n * T * D / (1 - D)
    print(f"\n{name}: n={dg.n} m={dg.m} ec {k} it {ec.solve_ms:.1f} ms, "
          f"fused {fu.trace.iterations} it {fu.solve_ms:.1f} ms")
    return ec, fu


def test_config3_rmat24_bfs_relabel():
    p = fb.RmatParams(24, 16, seed=3)
    with fb.DeviceGraph.generate_rmat(p, relabel_bfs=True) as dg:
        assert dg.validate() == 0
        assert dg.m == 263_434_595  # SURVEY probe: relabelling does not change m
        ec, _ = _properties(dg, "config3")
    # EC iteration counts are relabel-invariant; natural order = 61
    assert ec.trace.iterations == 61


def test_config4_chunglu():
    with fb.DeviceGraph.generate_chunglu(1 << 26, 1_200_000_000, seed=4) as dg:
        assert dg.validate() == 0
        assert dg.m > 500_000_000
        _properties(dg, "config4")


def test_config5_rmat28():
    with fb.DeviceGraph.generate_rmat(fb.RmatParams(28, 16, seed=5)) as dg:
        assert dg.validate() == 0
        assert 4_000_000_000 < dg.m < 4_294_967_296
        _properties(dg, "config5")


@pytest.mark.parametrize("config", ["4", "5"])
def test_pb_engines_full_size(config):
    """FPR_B200_OPT_PB at full size: the propagation-blocked EC gives the pull
    EC's iteration count and ranks within 1e-12 relative (the oracle's
    per-iteration bar, here against the oracle-checked pull engine); the
    FusEd schedule on PB sweeps converges in fewer sweeps to within the
    geometric-tail bound of the EC fixed point."""
    def make(**kw):
        if config == "4":
            return fb.DeviceGraph.generate_chunglu(1 << 26, 1_200_000_000, seed=4, **kw)
        return fb.DeviceGraph.generate_rmat(fb.RmatParams(28, 16, seed=5), **kw)

    cfg = fb.PageRankConfig(threshold=T)
    with make() as dg:
        ec = dg.run(fb.ENGINE_EC, cfg)
    with make(pb=True) as dg:
        pb = dg.run(fb.ENGINE_EC, cfg)
        ls = dg.run(fb.ENGINE_FUSED_LOCKSTEP, cfg)
        waves = len(dg.wave_starts()) - 1
        n = dg.n
    assert pb.trace.iterations == ec.trace.iterations and pb.trace.converged
    assert float(np.max(np.abs(pb.ranks.values - ec.ranks.values) / ec.ranks.values)) <= 1e-12
    assert ls.trace.converged and ls.trace.iterations < ec.trace.iterations
    assert fb.l1_norm(ls.ranks.values, ec.ranks.values) <= 2 * n * T * D / (1 - D)
    print(f"\nconfig{config} PB: ec {pb.trace.iterations} it {pb.solve_ms:.1f} ms, "
          f"lockstep ({waves} waves) {ls.trace.iterations} it {ls.solve_ms:.1f} ms")
