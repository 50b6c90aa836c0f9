"""Measurement probes (not part of the product; run on a B200 through gpurun).

  python scripts/probe.py sweep CONFIGS [--engines ec,fused,lockstep] [--sweep auto|pb|pull]
                                [--geoms 13:21,12:21] [--reorder degree|sources] [--reps 1]
      per-sweep device times, iterations, GTEPS and the BASELINE roofline
      fraction and a digest of the rank bits (compare variant builds); --geoms sets the propagation-blocked bin:chunk shifts; every
      PB run is repeated and checked bit-for-bit (fixed-order row sums).
  python scripts/probe.py waves CONFIG [--waves 1,2,4,8,16,32] [--sweep auto|pb|pull]
      the lockstep FusEd schedule's sweeps and time against its wave count.
  python scripts/probe.py once CONFIG [--engine ec] [--iters 2] [--sweep auto]
      one short resident solve: the target for ncu captures (profiles/).
  python scripts/probe.py e2e CONFIG
      create / run / destroy breakdown of the host-buffer path (fpr_b200_graph_create
      on pinned u64 arrays: upload + narrowing + partition, then the sweep
      layout on the first run).
  python scripts/probe.py ref CONFIG [--iters 1,2,3]
      the unmodified reference (oracle/_ref) on a device-generated graph:
      host RAM, graph hand-off + build_layout time, ec_par / fused_par per
      iteration on every host thread.

CONFIGS are BASELINE configs: 1 (R-MAT s16), 2 (uniform 2^22), 3 (R-MAT s24 +
BFS relabel), 4 (Chung-Lu 2^26), 5 (R-MAT s28).  FPR_B200_LIB=<path> selects a
variant build (make -C paper_2203_09284_b200/csrc variant / pbvariant).
"""
import argparse
import hashlib
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import paper_2203_09284_b200 as fb  # noqa: E402

PEAK = 6549.1
try:
    PEAK = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))["hbm_gbs"]
except Exception:
    pass
ENGINES = {"ec": fb.ENGINE_EC, "fused": fb.ENGINE_FUSED, "lockstep": fb.ENGINE_FUSED_LOCKSTEP}


def make(c, **kw):
    if c == "1":
        return fb.DeviceGraph.generate_rmat(fb.RmatParams(16, 16, seed=1), **kw)
    if c == "2":
        return fb.DeviceGraph.generate_uniform(1 << 22, 16, 2, **kw)
    if c == "3":
        return fb.DeviceGraph.generate_rmat(fb.RmatParams(24, 16, seed=3), relabel_bfs=True, **kw)
    if c == "4":
        return fb.DeviceGraph.generate_chunglu(1 << 26, 1_200_000_000, seed=4, **kw)
    return fb.DeviceGraph.generate_rmat(fb.RmatParams(28, 16, seed=5), **kw)


def sweep_kw(a):
    return {"pb": None if a.sweep == "auto" else a.sweep == "pb"}


def cmd_sweep(a):
    cfg = fb.PageRankConfig(threshold=1e-10)
    geoms = [g.split(":") for g in a.geoms.split(",")] if a.geoms else [None]
    for c in a.configs.split(","):
        for geom in geoms:
            if geom:
                os.environ["FPR_B200_PB_SHIFT"], os.environ["FPR_B200_PB_CHUNK_SHIFT"] = geom
            with make(c, reorder=a.reorder or False, **sweep_kw(a)) as dg:
                for e in a.engines.split(","):
                    t0 = time.perf_counter()
                    first = dg.run(ENGINES[e], fb.PageRankConfig(threshold=1e-10, max_iterations=1), copy_ranks=False)
                    t1 = time.perf_counter()
                    for _ in range(a.reps):
                        r = dg.run(ENGINES[e], cfg)
                    r2 = dg.run(ENGINES[e], cfg)
                    same = bool(np.array_equal(r.ranks.values.view(np.uint64), r2.ranks.values.view(np.uint64)))
                    ms = r.solve_ms / r.trace.iterations
                    dig = hashlib.sha1(r.ranks.values.view(np.uint64).tobytes()).hexdigest()[:16]
                    print(f"cfg{c} {e} sweep={'pb' if r.sweep else 'pull'} geom={':'.join(geom) if geom else '-'}: "
                          f"{r.trace.iterations} it, {ms:.3f} ms/sweep, {dg.m / ms / 1e6:.1f} GTEPS, roofline "
                          f"{(12 * dg.m + 36 * dg.n) / ms / 1e6 / PEAK:.3f}, first run (layout) "
                          f"{1e3 * (t1 - t0):.0f} ms, rerun bit-equal {same}, ranks sha1 {dig}", flush=True)


def cmd_waves(a):
    cfg = fb.PageRankConfig(threshold=1e-10)
    with make(a.configs, **sweep_kw(a)) as dg:
        for w in (int(x) for x in a.waves.split(",")):
            dg.set_wave_count(w)
            r = dg.run(fb.ENGINE_FUSED_LOCKSTEP, cfg, copy_ranks=False)
            print(f"cfg{a.configs} waves={w}: {r.trace.iterations} sweeps, "
                  f"{r.solve_ms / r.trace.iterations:.3f} ms/sweep, {r.solve_ms:.1f} ms", flush=True)


def cmd_once(a):
    with make(a.configs, **sweep_kw(a)) as dg:
        r = dg.run(ENGINES[a.engine], fb.PageRankConfig(threshold=1e-10, max_iterations=a.iters), copy_ranks=False)
        print(f"cfg{a.configs} {a.engine}: {r.trace.iterations} sweeps, {r.solve_ms / r.trace.iterations:.3f} "
              f"ms/sweep, m={dg.m}", flush=True)


def cmd_e2e(a):
    import torch

    with make(a.configs) as dg:
        n, m = dg.n, dg.m
        keep = [torch.empty(k, dtype=torch.int64, pin_memory=True) for k in (n + 1, m, n)]
        arrs = [t.numpy().view(np.uint64) for t in keep]
        dg.download_into(*arrs)
    pg = fb.Graph(n, m, *arrs)
    cfg = fb.PageRankConfig(threshold=1e-10)
    for _ in range(3):
        t0 = time.perf_counter()
        d = fb.DeviceGraph.from_graph(pg)
        t1 = time.perf_counter()
        r = d.run(fb.ENGINE_EC, cfg, copy_ranks=True, copy_trace=False)
        t2 = time.perf_counter()
        d.close()
        t3 = time.perf_counter()
        print(f"cfg{a.configs}: create {1e3 * (t1 - t0):.0f} ms, run {1e3 * (t2 - t1):.0f} ms (setup {r.setup_ms:.0f}, "
              f"solve {r.solve_ms:.0f}), destroy {1e3 * (t3 - t2):.0f} ms", flush=True)


def cmd_ref(a):
    from oracle import Graph as OGraph
    from oracle import load_reference

    mi = {l.split(":")[0]: int(l.split()[1]) * 1024 for l in open("/proc/meminfo")}
    threads = len(os.sched_getaffinity(0))
    print(json.dumps({"mem_total_gb": mi["MemTotal"] / 1e9, "mem_avail_gb": mi["MemAvailable"] / 1e9,
                      "threads": threads}), flush=True)
    ref = load_reference()
    with make(a.configs, pb=False) as dg:
        g = dg.download()
    og = OGraph(g.n, g.m, g.in_start, g.in_src, g.out_degree)
    t0 = time.perf_counter()
    h = ref.graph_handle(og)
    print(f"ref_graph_create (copy + build_layout) {time.perf_counter() - t0:.1f} s", flush=True)
    for k in (int(x) for x in a.iters_list.split(",")):
        for eng in ("ec_par", "fused_par"):
            r = ref.run(og, eng, 0.85, 1e-10, k, threads, handle=h)
            print(f"{eng} max_iter={k} T={threads}: {r.seconds:.2f} s", flush=True)
    ref.destroy(h)


def main():
    ap = argparse.ArgumentParser()
    sub = ap.add_subparsers(dest="cmd", required=True)
    for name in ("sweep", "waves", "once", "e2e", "ref"):
        p = sub.add_parser(name)
        p.add_argument("configs")
        p.add_argument("--sweep", default="auto", choices=["auto", "pb", "pull"])
        p.add_argument("--engines", default="ec")
        p.add_argument("--engine", default="ec")
        p.add_argument("--geoms", default="")
        p.add_argument("--reorder", default="")
        p.add_argument("--reps", type=int, default=1)
        p.add_argument("--waves", default="1,2,4,8,16,32")
        p.add_argument("--iters", type=int, default=2)
        p.add_argument("--iters-list", dest="iters_list", default="1,2,3")
    a = ap.parse_args()
    {"sweep": cmd_sweep, "waves": cmd_waves, "once": cmd_once, "e2e": cmd_e2e, "ref": cmd_ref}[a.cmd](a)


if __name__ == "__main__":
    main()
