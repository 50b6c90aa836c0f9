"""CPU checks of the oracle's restatements for the generators the reference
lacks (config 3's BFS relabel, config 4's Chung-Lu): hand-checked
small cases and invariants.  No GPU."""
import numpy as np

from golden_util import load


def test_bfs_relabel_hand_case(oracle):
    # 0->2, 0->1, 2->3, 1->3, 3->0, 4 isolated, 5->4
    src = np.array([0, 0, 2, 1, 3, 5], np.uint64)
    dst = np.array([2, 1, 3, 3, 0, 4], np.uint64)
    g = oracle.build_csr(6, src, dst)
    new = oracle.bfs_relabel(g, 0)
    # BFS from 0: neighbours ascending -> 1, 2; then 1's 3; unreached 4, 5 ascending
    assert new.tolist() == [0, 1, 2, 3, 4, 5]
    new2 = oracle.bfs_relabel(g, 5)
    # from 5: 5->4 (4 has no out-edges); unreached 0,1,2,3 appended ascending
    assert new2.tolist() == [2, 3, 4, 5, 1, 0]


def test_bfs_relabel_is_permutation_and_invariant(oracle):
    rec = load("rmat_s12_seed7.json")
    n, s, d = oracle.generate_rmat(12, 16, seed=7)
    g = oracle.build_csr(n, s, d)
    new = oracle.bfs_relabel(g, 0)
    assert np.array_equal(np.sort(new), np.arange(n, dtype=np.uint64))
    assert new[0] == 0
    r = oracle.relabel(g, new)
    assert r.m == g.m == rec["graph"]["m"]
    # EC iteration count is relabel-invariant (SURVEY §8(d) config 3 sanity check)
    a = oracle.pagerank_ec(g, threshold=1e-10)
    b = oracle.pagerank_ec(r, threshold=1e-10)
    assert a.iterations == b.iterations
    assert np.max(np.abs(b.ranks[new.astype(np.int64)] - a.ranks) / a.ranks) < 1e-12


def test_chunglu_definition(oracle):
    cdf = oracle.chunglu_cdf(2.1, 1000)
    assert np.all(np.diff(cdf) > 0) and abs(cdf[-1] - 1.0) < 1e-12
    n, s, d = oracle.generate_chunglu(1 << 12, 1 << 15, seed=4, kmax=1000)
    assert s.max() < n and d.max() < n
    n2, s2, d2 = oracle.generate_chunglu(1 << 12, 1 << 15, seed=4, kmax=1000)
    assert np.array_equal(s, s2) and np.array_equal(d, d2)
    g = oracle.build_csr(n, s, d)
    deg = g.out_degree + np.diff(g.in_start)
    # heavy tail: max degree far above the mean
    assert deg.max() > 10 * deg.mean()
