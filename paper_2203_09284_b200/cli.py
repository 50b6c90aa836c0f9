"""fpr-b200: the reference's missing bench CLI over the B200
engines.  Subcommands run / bench / gen / compare; CSV schema and exit codes
as specified (0 ok, 1 usage, 2 I/O, 3 non-convergence).

Graph sources:
  --graph PATH.fprg           FPRG cache (graph_cache.hpp format)
  --rmat SCALE:EF:SEED        fpr::generate_rmat (+ build_csr) on the device
  --rmat-bfs SCALE:EF:SEED    ... relabelled in BFS crawl order (config 3)
  --uniform N:DEG:SEED        testutil::random_sparse semantics (config 2)
  --chunglu N:DRAWS:SEED      config 4
  --edges PATH                SNAP edge-list text, parsed on the device
                              (build_csr(parse_edge_list(file)), edge_list.hpp)

Engines: ec_b200, fused_b200, fused_lockstep_b200.  The L1 reference column
(l1_vs_seq_ec) is taken from ec_b200, which equals the reference's ec_seq
within 1e-12 relative per iteration (tests/test_gpu_engines.py).
"""
from __future__ import annotations

import argparse
import csv
import io
import json
import sys
import time

import numpy as np

from . import (B200Error, DeviceGraph, EdgeSet, EngineKind, NORM_L1, NORM_LINF, PageRankConfig, ParseError,
               RmatParams, generate_edges, l1_norm, parse_engine, write_edge_list, ENGINE_EC, ENGINE_FUSED,
               ENGINE_FUSED_LOCKSTEP)
from .cache import CacheError, load_cache, save_cache

EXIT_OK, EXIT_USAGE, EXIT_IO, EXIT_NONCONV = 0, 1, 2, 3
CSV_COLUMNS = ["graph", "engine", "threshold", "threads", "iterations", "wall_time_s",
               "l1_vs_seq_ec", "converged"]
_ENGINES = {EngineKind.EcB200: ENGINE_EC, EngineKind.FusedB200: ENGINE_FUSED,
            EngineKind.FusedLockstepB200: ENGINE_FUSED_LOCKSTEP}


class UsageError(Exception):
    pass


def _triple(text: str, name: str) -> tuple[int, int, int]:
    try:
        a, b, c = (int(x) for x in text.split(":"))
        return a, b, c
    except ValueError:
        raise UsageError(f"--{name} expects A:B:C integers, got '{text}'")


def open_graph(args, norm=NORM_LINF) -> tuple[DeviceGraph, str]:
    given = [k for k in ("graph", "rmat", "rmat_bfs", "uniform", "chunglu", "edges") if getattr(args, k, None)]
    if len(given) != 1:
        raise UsageError("exactly one graph source is required "
                         "(--graph/--rmat/--rmat-bfs/--uniform/--chunglu/--edges)")
    k = given[0]
    v = getattr(args, k)
    # library options: internal renumbering,
    # propagation-blocked sweeps, lockstep waves per sweep
    ro = getattr(args, "reorder", "none")
    kw = {"norm": norm, "reorder": False if ro == "none" else ro, "pb": True if getattr(args, "pb", False) else None,
          "wave_count": int(getattr(args, "waves", 0))}
    if k == "graph":
        g = load_cache(v)  # CacheError -> I/O exit code
        return DeviceGraph.from_graph(g, **kw), v
    if k == "edges":
        text = np.fromfile(v, dtype=np.uint8)  # OSError -> I/O exit code
        return DeviceGraph.from_edge_list(text, **kw), v
    a, b, c = _triple(v, k.replace("_", "-"))
    if k in ("rmat", "rmat_bfs"):
        return DeviceGraph.generate_rmat(RmatParams(scale=a, edge_factor=b, seed=c),
                                         relabel_bfs=(k == "rmat_bfs"), **kw), f"{k}:{v}"
    if k == "uniform":
        return DeviceGraph.generate_uniform(a, b, c, **kw), f"uniform:{v}"
    return DeviceGraph.generate_chunglu(a, b, c, **kw), f"chunglu:{v}"


def _engine(tag: str) -> int:
    kind = parse_engine(tag)
    if kind not in _ENGINES:
        raise UsageError(f"engine '{tag}' is a reference CPU engine; this CLI runs "
                         + "|".join(k.value for k in _ENGINES))
    return _ENGINES[kind]


def _threads(args) -> list[int]:
    """--threads N or a comma list (bench sweeps every value; SPEC BenchSpec)."""
    try:
        ts = [int(x) for x in str(args.threads).split(",") if x.strip()]
    except ValueError:
        raise UsageError(f"--threads expects integers, got '{args.threads}'")
    if not ts or min(ts) < 1:
        raise UsageError("--threads values must be positive")
    return ts


def _cfg(args, threshold=None, threads=None) -> PageRankConfig:
    return PageRankConfig(damping=args.damping, threshold=threshold if threshold is not None else args.threshold,
                          max_iterations=args.max_iters,
                          thread_count=threads if threads is not None else _threads(args)[0])


def cmd_run(args, out) -> int:
    engine = _engine(args.engine)  # usage errors before any device work
    dg, label = open_graph(args)
    with dg:
        t0 = time.perf_counter()
        r = dg.run(engine, _cfg(args))
        wall = time.perf_counter() - t0
    vals = r.ranks.values
    order = sorted(range(len(vals)), key=lambda i: (-vals[i], i))[: args.topk]  # ties: ascending id
    out.write(f"graph={label} engine={args.engine} iterations={r.trace.iterations} "
              f"wall_time_s={wall:.6f} solve_ms={r.solve_ms:.3f} converged={str(r.trace.converged).lower()}\n")
    out.write(", ".join(f"{i}:{vals[i]:.17g}" for i in order) + "\n")
    return EXIT_OK if r.trace.converged else EXIT_NONCONV


def cmd_bench(args, out) -> int:
    engines = [e.strip() for e in args.engines.split(",") if e.strip()]
    thresholds = [float(t) for t in args.thresholds.split(",")]
    threads = _threads(args)
    if not engines or not thresholds:
        raise UsageError("bench needs at least one engine and one threshold")
    for e in engines:
        _engine(e)
    dg, label = open_graph(args)
    rows = []
    with dg:
        # engines x thresholds x threads x reps (SPEC cmd_bench); the GPU
        # engines validate thread_count and otherwise ignore it
        for t in thresholds:
            try:
                ref = dg.run(ENGINE_EC, _cfg(args, t))  # the L1 reference, run first
            except (B200Error, ValueError):
                ref = None
            for e in engines:
                for th in threads:
                    best, res = None, None
                    try:
                        for _ in range(max(1, args.reps)):  # min over repetitions
                            t0 = time.perf_counter()
                            r = dg.run(_engine(e), _cfg(args, t, th))
                            w = time.perf_counter() - t0
                            if best is None or w < best:
                                best, res = w, r
                    except (B200Error, ValueError) as ex:  # a failed cell is a row, not an abort
                        sys.stderr.write(f"fpr-b200: {e} at threshold {t!r}: {ex}\n")
                        rows.append({"graph": label, "engine": e, "threshold": repr(t), "threads": th,
                                     "iterations": 0, "wall_time_s": "", "l1_vs_seq_ec": "", "converged": "false"})
                        continue
                    l1 = repr(l1_norm(res.ranks.values, ref.ranks.values)) if ref is not None else ""
                    rows.append({"graph": label, "engine": e, "threshold": repr(t), "threads": th,
                                 "iterations": res.trace.iterations, "wall_time_s": f"{best:.6f}",
                                 "l1_vs_seq_ec": l1, "converged": str(res.trace.converged).lower()})
    if args.format == "json":
        out.write(json.dumps(rows) + "\n")
    else:
        w = csv.DictWriter(out, fieldnames=CSV_COLUMNS, lineterminator="\n")
        w.writeheader()
        w.writerows(rows)
    return EXIT_OK


def cmd_gen(args, out) -> int:
    """SPEC cmd_gen: the GENERATED EdgeSet as SNAP text -- header comment lines
    with the parameters and seed, then one "src dst" line per draw in
    generation order (--rmat: generate_rmat's draws, self-loops and duplicates
    kept; --uniform: random_sparse's kept draws).  --format fprg writes the
    normalised graph (build_csr of it) as an FPRG cache instead; other graph
    sources have no generated EdgeSet and write their normalised edges."""
    if args.reorder != "none":
        raise UsageError("gen writes the graph in the caller's ids; --reorder applies to run/bench")
    src_kind = "rmat" if args.rmat else ("uniform" if args.uniform else None)
    if args.format == "edges" and src_kind:
        a, b, c = _triple(args.rmat or args.uniform, src_kind)
        if src_kind == "rmat":
            p = RmatParams(scale=a, edge_factor=b, seed=c)
            es = generate_edges("rmat", params=p)
            header = [f"fpr-b200 gen: generate_rmat scale={a} edge_factor={b} a={p.a} b={p.b} c={p.c} d={p.d}",
                      f"seed={c} n={es.n} edges={len(es.edges)}"]
        else:
            es = generate_edges("uniform", n=a, avg_degree=b, seed=c)
            header = [f"fpr-b200 gen: random_sparse n={a} avg_degree={b}",
                      f"seed={c} n={es.n} edges={len(es.edges)}"]
        with open(args.out, "wb") as f:
            f.write(write_edge_list(es, header))
        out.write(f"wrote {args.out}: {src_kind}:{a}:{b}:{c} n={es.n} edges={len(es.edges)}\n")
        return EXIT_OK
    dg, label = open_graph(args)
    with dg:
        g = dg.download()
    if args.format == "edges":  # no generator EdgeSet: the normalised graph's edges
        dst = np.repeat(np.arange(g.n, dtype=np.uint64), np.diff(g.in_start.astype(np.int64)))
        text = write_edge_list(EdgeSet(g.n, np.stack([g.in_src, dst], axis=1)),
                               [f"fpr-b200 gen: {label} (normalised: build_csr) n={g.n} m={g.m}"])
        with open(args.out, "wb") as f:
            f.write(text)
    else:
        save_cache(g, args.out)  # FPRG (graph_cache.hpp); CacheError -> I/O
    out.write(f"wrote {args.out}: {label} n={g.n} m={g.m}\n")
    return EXIT_OK


def cmd_compare(args, out) -> int:
    dg, label = open_graph(args)
    traces, ranks = {}, {}
    with dg:
        for kind in _ENGINES:
            r = dg.run(_ENGINES[kind], _cfg(args))
            traces[kind.value], ranks[kind.value] = r.trace.errors, r.ranks.values
    names = list(traces)
    w = csv.writer(out, lineterminator="\n")
    w.writerow(["iteration"] + names)
    for i in range(max(len(t) for t in traces.values())):
        w.writerow([i + 1] + [repr(float(traces[n][i])) if i < len(traces[n]) else "" for n in names])
    out.write("\n")
    w.writerow(["l1"] + names)
    for a in names:
        w.writerow([a] + [repr(l1_norm(ranks[a], ranks[b])) for b in names])
    return EXIT_OK


def build_parser() -> argparse.ArgumentParser:
    ap = argparse.ArgumentParser(prog="fpr-b200", description=__doc__.split("\n")[0])
    sub = ap.add_subparsers(dest="cmd", required=True)

    def common(p):
        p.add_argument("--graph")
        p.add_argument("--rmat")
        p.add_argument("--rmat-bfs", dest="rmat_bfs")
        p.add_argument("--uniform")
        p.add_argument("--chunglu")
        p.add_argument("--edges")
        p.add_argument("--damping", type=float, default=0.85)
        p.add_argument("--threshold", type=float, default=1e-15)
        p.add_argument("--threads", default="1", help="N, or a comma list (bench sweeps them)")
        p.add_argument("--max-iters", dest="max_iters", type=int, default=10000)
        p.add_argument("--reorder", choices=["none", "degree", "sources"], default="none",
                       help="internal renumbering (FPR_B200_OPT_REORDER / _REORDER_SOURCES)")
        p.add_argument("--pb", action="store_true",
                       help="force propagation-blocked sweeps (FPR_B200_OPT_PB; default: the library picks)")
        p.add_argument("--waves", type=int, default=0, help="lockstep waves per sweep (0 = auto)")

    p = sub.add_parser("run")
    common(p)
    p.add_argument("--engine", default="ec_b200")
    p.add_argument("--topk", type=int, default=10)
    p = sub.add_parser("bench")
    common(p)
    p.add_argument("--engines", default="ec_b200,fused_b200")
    p.add_argument("--thresholds", default="1e-8,1e-12")
    p.add_argument("--reps", type=int, default=1)
    p.add_argument("--format", choices=["csv", "json"], default="csv")
    p.add_argument("--out")
    p = sub.add_parser("gen")
    common(p)
    p.add_argument("--out", required=True)
    p.add_argument("--format", choices=["edges", "fprg"], default="edges",
                   help="edges: SNAP text of the generated EdgeSet (SPEC cmd_gen); fprg: the normalised graph")
    p = sub.add_parser("compare")
    common(p)
    return ap


def main(argv=None, out=None) -> int:
    out = out or sys.stdout
    try:
        args = build_parser().parse_args(argv)
    except SystemExit as e:
        return EXIT_USAGE if e.code else EXIT_OK
    try:
        buf = io.StringIO() if getattr(args, "out", None) and args.cmd == "bench" else out
        rc = {"run": cmd_run, "bench": cmd_bench, "gen": cmd_gen, "compare": cmd_compare}[args.cmd](args, buf)
        if buf is not out:
            try:
                with open(args.out, "w") as f:
                    f.write(buf.getvalue())
            except OSError as e:
                sys.stderr.write(f"fpr-b200: cannot write {args.out}: {e}\n")
                return EXIT_IO
        return rc
    except UsageError as e:
        sys.stderr.write(f"fpr-b200: {e}\n")
        return EXIT_USAGE
    except (CacheError, OSError, ParseError) as e:  # a malformed input file is an I/O error
        sys.stderr.write(f"fpr-b200: {e}\n")
        return EXIT_IO
    except ValueError as e:  # reference validation messages (invalid_argument)
        sys.stderr.write(f"fpr-b200: {e}\n")
        return EXIT_USAGE


if __name__ == "__main__":
    sys.exit(main())
