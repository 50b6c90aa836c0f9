"""EC ms/iter with FPR_B200_OPT_PB against the plain pull engine:
python scripts/pb_probe.py [configs]  (env GEOMS="13:20,12:20,13:19" = shift:chunk_shift pairs;
PB_ONLY=1 skips the plain pull run)."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_2203_09284_b200 as fb

cfg = fb.PageRankConfig(threshold=1e-10)


def make(c, **kw):
    if c.startswith("2"):
        return fb.DeviceGraph.generate_uniform(1 << 22, 16, 2, **kw)
    if c.startswith("3"):
        return fb.DeviceGraph.generate_rmat(fb.RmatParams(24, 16, seed=3), relabel_bfs=True, **kw)
    if c.startswith("4"):
        return fb.DeviceGraph.generate_chunglu(1 << 26, 1_200_000_000, seed=4, **kw)
    return fb.DeviceGraph.generate_rmat(fb.RmatParams(28, 16, seed=5), **kw)


def main():
    geoms = [tuple(int(v) for v in x.split(":")) for x in os.environ.get("GEOMS", "13:21").split(",")]
    for c in (sys.argv[1:] or ["2", "4", "5"]):
        reorder = c.endswith("r")
        plain = None
        if not os.environ.get("PB_ONLY"):
            with make(c, reorder=reorder) as dg:
                r = dg.run(fb.ENGINE_EC, cfg, copy_ranks=True)
                plain = r.ranks.values
                ms = r.solve_ms / r.trace.iterations
                print(f"cfg{c} plain: {r.trace.iterations} it, {ms:.3f} ms/it, {dg.m / ms / 1e6:.1f} GTEPS", flush=True)
        for sh, cs in geoms:
            os.environ["FPR_B200_PB_SHIFT"] = str(sh)
            os.environ["FPR_B200_PB_CHUNK_SHIFT"] = str(cs)
            with make(c, reorder=reorder, pb=True) as dg:
                t0 = time.perf_counter()
                dg.run(fb.ENGINE_EC, fb.PageRankConfig(threshold=1e-10, max_iterations=1), copy_ranks=False)
                t1 = time.perf_counter()
                r = dg.run(fb.ENGINE_EC, cfg, copy_ranks=True)
                r2 = dg.run(fb.ENGINE_EC, cfg, copy_ranks=True)
                same = bool(np.array_equal(r.ranks.values.view(np.uint64), r2.ranks.values.view(np.uint64))
                            and np.array_equal(r.trace.errors, r2.trace.errors))
                ms = r.solve_ms / r.trace.iterations
                d = np.max(np.abs(r.ranks.values - plain) / plain) if plain is not None else float("nan")
                per = ", ".join(f"{x / 1e6:.2f}" for x in r.trace.iter_ns[: r.trace.iterations])
                print(f"cfg{c} pb {sh}:{cs}: {r.trace.iterations} it, {ms:.3f} ms/it, {dg.m / ms / 1e6:.1f} GTEPS, "
                      f"build+1 sweep {1e3 * (t1 - t0):.0f} ms, max rel vs plain {d:.2e}, rerun bit-equal {same}; per-iter ms [{per}]",
                      flush=True)


if __name__ == "__main__":
    main()
