"""Regenerate tests/golden/*.json from the REFERENCE ITSELF.

Runs only in the build container, where /root/reference exists and
oracle/_ref/libfpr_ref.so has been compiled from the unmodified reference
headers (``make -C oracle``).  Every number in the fixtures is produced by a
reference function (generate_rmat, testutil::random_sparse, build_csr,
pagerank_{ec,fused}_seq, pagerank_dense_oracle) -- never by this repo's code.

    python tests/golden/make_golden.py            # all fixtures
    python tests/golden/make_golden.py --skip-config2
    python tests/golden/make_golden.py --only edge_list

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
sys.path.insert(0, os.path.join(ROOT, "tests"))
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


def edge_list_fixture(ref: Reference) -> dict:
    """fpr::parse_edge_list (edge_list.hpp:39-80) on the inputs of the
    reference's own tests (io_ingest_test.cpp:25-93), edge cases, seeded fuzz
    texts and a large sparse-id text (digests only)."""
    from golden_util import fuzz_text, roundtrip_texts, sparse_text_from_edges

    named = [
        ("SkipsCommentsAndParses", b"# comment\n0 1\n1 2\n"),
        ("CompactsSparseIds", b"5 9\n9 5\n"),
        ("RejectsMalformedLine", b"0 x\n"),
        ("RejectsOverflowingToken", b"0 1\n99999999999999999999999 2\n"),
        ("RejectsTrailingGarbage", b"0 1 2\n"),
        ("RejectsShortLine", b"0\n"),
        ("RejectsNegative", b"0 -1\n"),
        ("SkipsBlankAndPercentLines", b"% header\n\n   \n0 1\n"),
        ("empty", b""),
        ("only_comments", b"# a\n% b\n\n"),
        ("no_final_newline", b"3 4\n4 5"),
        ("crlf_tabs", b"1\t2\r\n3 \t 4\r\n"),
        ("indented_hash_is_a_token", b"  # x\n"),
        ("u64_max_then_overflow", b"18446744073709551615 0\n18446744073709551616 1\n"),
        ("vertical_tab_not_whitespace", b"\x0b1 2\n"),
        ("form_feed_not_whitespace", b"1 2\x0c\n"),
        ("leading_zeros", b"007 0007\n7 0\n"),
        ("plus_sign", b"+1 2\n"),
        ("trailing_whitespace_and_blank_tail", b"1 2 \t\r\n\n\n"),
        ("self_loops_kept", b"4 4\n4 5\n"),
        ("first_error_wins", b"1 2\n3\n4 x\n"),
        ("nul_byte", b"1 2\n3\x004\n"),
        ("long_line", b"1 " + b"9" * 19 + b"\n" + b"2 " + b" " * 5000 + b"3\n"),
    ]
    named += [(f"RenderRoundTrip_{i}", t) for i, t in enumerate(roundtrip_texts())]
    named += [(f"fuzz_{s}", fuzz_text(s, 1 + s % 60, bad_rate=0.02 if s % 3 == 0 else 0.0))
              for s in range(120)]
    cases = []
    for name, text in named:
        p = ref.parse_edge_list(text)
        cases.append({"name": name, "text": text.decode("latin-1"), "n": p.n,
                      "edges": p.edges.reshape(-1).tolist(), "error_line": p.error_line, "error": p.error})
    # large: RMAT(12, 16, 7) draws as sparse ids with comment lines
    _, s, d = ref.generate_rmat(12, 16, seed=7)
    text = sparse_text_from_edges(s, d)
    p = ref.parse_edge_list(text)
    large = {"source": "generate_rmat(12,16,seed=7) draws, raw = id*2654435761+12345, '# block' every 1000",
             "bytes": len(text), "text_sha256": hashlib.sha256(text).hexdigest(), "n": p.n,
             "m": int(len(p.edges)), "edges_sha256": sha(p.edges.reshape(-1))}
    g = ref.build_csr(p.n, p.edges[:, 0], p.edges[:, 1])
    large["graph"] = graph_digest(g)
    return {"cases": cases, "large": large}


def config3_fixture(ref: Reference, sample=4096) -> dict:
    """BASELINE config 3: generate_rmat(24, 16, seed 3) -> build_csr, BFS
    crawl-order relabel, build_csr again -- every array by the reference,
    except the BFS permutation itself (the reference has no relabel; it is
    SURVEY §8(d)'s definition, restated by fo_bfs_relabel and pinned against
    the device relabel in tests/test_gpu_generate.py).  Then the reference's
    pagerank_ec_seq and pagerank_fused_seq at 1e-10 (L-inf): iteration
    counts, every iteration's error (hex) and `sample` seeded rank samples.
    About 15 minutes on 8 cores (ec_seq 61 x ~7 s, fused_seq 41 x ~7 s)."""
    import time

    from oracle import Oracle

    t0 = time.time()
    n, s, d = ref.generate_rmat(24, 16, seed=3)
    rec = {"params": {"scale": 24, "edge_factor": 16, "a": 0.57, "b": 0.19, "c": 0.19, "d": 0.05, "seed": 3,
                      "relabel": "bfs from old id 0 (SURVEY §8(d))"},
           "draws_sha256": {"src": sha(s), "dst": sha(d)}}
    g0 = ref.build_csr(n, s, d)
    del s, d
    rec["graph_natural"] = graph_digest(g0)
    new_id = Oracle().bfs_relabel(g0, 0)
    rec["bfs_new_id_sha256"] = sha(new_id)
    dst = np.repeat(np.arange(g0.n, dtype=np.uint64), np.diff(g0.in_start).astype(np.int64))
    g = ref.build_csr(n, new_id[g0.in_src], new_id[dst])
    del g0, dst, new_id
    rec["graph"] = graph_digest(g)
    print(f"config3 graph built in {time.time() - t0:.0f} s", flush=True)
    idx = np.sort(np.random.default_rng(3).choice(n, size=sample, replace=False))
    rec["runs"] = {}
    h = ref.graph_handle(g)
    try:
        for eng in ("ec_seq", "fused_seq"):
            t1 = time.time()
            r = ref.run(g, eng, threshold=1e-10, handle=h)
            rec["runs"][f"{eng}@1e-10"] = run_digest(r, idx)
            rec["runs"][f"{eng}@1e-10"]["seconds"] = r.seconds
            print(f"config3 {eng}: {r.iterations} iterations, {time.time() - t1:.0f} s", flush=True)
    finally:
        ref.destroy(h)
    return rec


def main() -> None:
    ap = argparse.ArgumentParser()
    ap.add_argument("--skip-config2", action="store_true")
    ap.add_argument("--only", choices=["edge_list", "config3"], help="regenerate one fixture")
    args = ap.parse_args()
    ref = Reference()
    if args.only == "edge_list":
        json.dump(edge_list_fixture(ref), open(os.path.join(OUT, "edge_list.json"), "w"), indent=0)
        return
    if args.only == "config3":
        json.dump(config3_fixture(ref), open(os.path.join(OUT, "config3.json"), "w"), indent=1)
        return

    json.dump(kats(ref), open(os.path.join(OUT, "kat.json"), "w"), indent=1)
    json.dump(corpus(ref), open(os.path.join(OUT, "corpus.json"), "w"))

    # io_ingest_test.cpp:143-155 regression pin (max_in == 343) + full digests.
    json.dump(rmat_fixture(ref, 10, 16, 42, [1e-10]), open(os.path.join(OUT, "rmat_s10_seed42.json"), "w"), indent=1)
    # SPEC AC4 graph RMAT(12,16,7) across the threshold sweep.
    json.dump(rmat_fixture(ref, 12, 16, 7, [1e-6, 1e-8, 1e-10, 1e-12]),
              open(os.path.join(OUT, "rmat_s12_seed7.json"), "w"), indent=1)
    # BASELINE config 1.
    json.dump(rmat_fixture(ref, 16, 16, 1, [1e-10, 1e-13]), open(os.path.join(OUT, "config1.json"), "w"), indent=1)

    json.dump(edge_list_fixture(ref), open(os.path.join(OUT, "edge_list.json"), "w"), indent=0)

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
