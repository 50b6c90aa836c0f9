"""Regenerate tests/golden/*.json from the REFERENCE ITSELF.

Runs only in the build container, where /root/reference exists and
oracle/_ref/libfpr_ref.so has been compiled from the unmodified reference
headers (``make -C oracle``).  Every number in the fixtures is produced by a
reference function (generate_rmat, testutil::random_sparse, build_csr,
pagerank_{ec,fused}_seq, pagerank_dense_oracle) -- never by this repo's code.

    python tests/golden/make_golden.py            # all fixtures
    python tests/golden/make_golden.py --skip-config2

The fixtures pin the C restatement (oracle/fpr_oracle.c) bit-exactly in
tests/test_oracle.py, and give the GPU parity tests reference answers that do
not need /root/reference at run time.
"""
from __future__ import annotations

import argparse
import hashlib
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
from oracle import Graph, Reference  # noqa: E402

OUT = os.path.dirname(os.path.abspath(__file__))


def sha(a: np.ndarray) -> str:
    return hashlib.sha256(np.ascontiguousarray(a).astype("<" + a.dtype.str[1:]).tobytes()).hexdigest()


def hexes(a) -> list[str]:
    return [float(x).hex() for x in a]


def graph_digest(g: Graph) -> dict:
    return {"n": g.n, "m": g.m, "in_start": sha(g.in_start), "in_src": sha(g.in_src),
            "out_degree": sha(g.out_degree), "max_in": int(np.diff(g.in_start).max()),
            "dangling": int((g.out_degree == 0).sum()),
            "zero_in": int((np.diff(g.in_start) == 0).sum())}


def run_digest(r, sample_idx) -> dict:
    return {"iterations": r.iterations, "errors": hexes(r.errors), "ranks_sha256": sha(r.ranks),
            "ranks_sum": float(r.ranks.sum()).hex(),
            "sample": {int(i): float(r.ranks[i]).hex() for i in sample_idx}}


def small_graph(n, edges) -> tuple[int, np.ndarray, np.ndarray]:
    e = np.array(edges, dtype=np.uint64).reshape(-1, 2)
    return n, e[:, 0].copy(), e[:, 1].copy()


def kats(ref: Reference) -> dict:
    """SPEC.md examples: gather_ranks_jacobi :208-211, pagerank_ec_seq :218-221."""
    cases = {
        "two_cycle": (2, [(0, 1), (1, 0)]),
        "single_dangling": (1, []),
        "three_vertex": (3, [(0, 2), (1, 2), (2, 0), (2, 1)]),
        "star": (5, [(1, 0), (2, 0), (3, 0), (4, 0), (0, 1)]),
        "loops_and_dups": (4, [(0, 1), (0, 1), (1, 1), (1, 2), (2, 3), (3, 0), (3, 0), (2, 2)]),
    }
    out = {}
    for name, (n, edges) in cases.items():
        g = ref.build_csr(*small_graph(n, edges))
        rec = {"n": n, "edges": edges, "m": g.m, "in_start": g.in_start.tolist(),
               "in_src": g.in_src.tolist(), "out_degree": g.out_degree.tolist()}
        for eng in ("ec_seq", "fused_seq"):
            r = ref.run(g, eng, threshold=1e-15)
            rec[eng] = {"iterations": r.iterations, "ranks": hexes(r.ranks), "errors": hexes(r.errors)}
        one = ref.run(g, "ec_seq", threshold=1e-15, max_iterations=1)
        rec["ec_one_step"] = hexes(one.ranks)
        rec["dense"] = hexes(ref.dense_oracle(g, threshold=1e-15))
        out[name] = rec
    return out


def corpus(ref: Reference, count=200, seed=20220318) -> list:
    """SPEC.md AC1 corpus shape: n in [1,16], density in {0.1,0.3,0.6}, dangling allowed.
    The edge lists are drawn here with numpy (the reference's testutil Bernoulli
    generator is not exported); every result is the reference's."""
    rng = np.random.default_rng(seed)
    out = []
    for k in range(count):
        n = int(rng.integers(1, 17))
        dens = [0.1, 0.3, 0.6][k % 3]
        mask = rng.random((n, n)) < dens
        np.fill_diagonal(mask, False)
        edges = [(int(u), int(v)) for u, v in zip(*np.nonzero(mask))]
        g = ref.build_csr(*small_graph(n, edges))
        ec = ref.run(g, "ec_seq", threshold=1e-13)
        fu = ref.run(g, "fused_seq", threshold=1e-13)
        dn = ref.dense_oracle(g, threshold=1e-13)
        out.append({"n": n, "density": dens, "edges": edges,
                    "ec_seq": {"iterations": ec.iterations, "ranks": hexes(ec.ranks)},
                    "fused_seq": {"iterations": fu.iterations, "ranks": hexes(fu.ranks)},
                    "dense": hexes(dn)})
    return out


def rmat_fixture(ref: Reference, scale, ef, seed, thresholds, sample=64) -> dict:
    n, s, d = ref.generate_rmat(scale, ef, seed=seed)
    g = ref.build_csr(n, s, d)
    rng = np.random.default_rng(seed)
    idx = np.sort(rng.choice(n, size=min(sample, n), replace=False))
    rec = {"params": {"scale": scale, "edge_factor": ef, "a": 0.57, "b": 0.19, "c": 0.19,
                      "d": 0.05, "seed": seed},
           "draws_sha256": {"src": sha(s), "dst": sha(d)}, "graph": graph_digest(g), "runs": {}}
    h = ref.graph_handle(g)
    try:
        for t in thresholds:
            for eng in ("ec_seq", "fused_seq"):
                r = ref.run(g, eng, threshold=t, handle=h)
                rec["runs"][f"{eng}@{t:g}"] = run_digest(r, idx)
    finally:
        ref.destroy(h)
    return rec


def main() -> None:
    ap = argparse.ArgumentParser()
    ap.add_argument("--skip-config2", action="store_true")
    args = ap.parse_args()
    ref = Reference()

    json.dump(kats(ref), open(os.path.join(OUT, "kat.json"), "w"), indent=1)
    json.dump(corpus(ref), open(os.path.join(OUT, "corpus.json"), "w"))

    # io_ingest_test.cpp:143-155 regression pin (max_in == 343) + full digests.
    json.dump(rmat_fixture(ref, 10, 16, 42, [1e-10]), open(os.path.join(OUT, "rmat_s10_seed42.json"), "w"), indent=1)
    # SPEC AC4 graph RMAT(12,16,7) across the threshold sweep.
    json.dump(rmat_fixture(ref, 12, 16, 7, [1e-6, 1e-8, 1e-10, 1e-12]),
              open(os.path.join(OUT, "rmat_s12_seed7.json"), "w"), indent=1)
    # BASELINE config 1.
    json.dump(rmat_fixture(ref, 16, 16, 1, [1e-10, 1e-13]), open(os.path.join(OUT, "config1.json"), "w"), indent=1)

    if not args.skip_config2:
        # BASELINE config 2: random_sparse(n=2^22, avg_degree=16, SplitMix64(2)) semantics.
        n, s, d = ref.random_sparse(1 << 22, 16, 2)
        g = ref.build_csr(n, s, d)
        idx = np.sort(np.random.default_rng(2).choice(n, size=64, replace=False))
        rec = {"params": {"n": n, "avg_degree": 16, "seed": 2}, "kept_draws": len(s),
               "draws_sha256": {"src": sha(s), "dst": sha(d)}, "graph": graph_digest(g), "runs": {}}
        h = ref.graph_handle(g)
        try:
            for eng in ("ec_seq", "fused_seq"):
                r = ref.run(g, eng, threshold=1e-10, handle=h)
                rec["runs"][f"{eng}@1e-10"] = run_digest(r, idx)
        finally:
            ref.destroy(h)
        json.dump(rec, open(os.path.join(OUT, "config2.json"), "w"), indent=1)
    print("golden fixtures written to", OUT)


if __name__ == "__main__":
    main()
