"""EC ms/iter with and without FPR_B200_OPT_BLOCKED on configs 2-5: python scripts/blocked_probe.py [configs] (env FPR_B200_BLOCK_SHIFT)."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_2203_09284_b200 as fb
cfg = fb.PageRankConfig(threshold=1e-10)
shifts = [int(x) for x in os.environ.get("SHIFTS", "22").split(",")]
for c in (sys.argv[1:] or ["3", "4", "5"]):
    for reorder in (False, True):
        kw = dict(reorder=reorder, blocked=True)
        if c == "2":
            dg = fb.DeviceGraph.generate_uniform(1 << 22, 16, 2, **kw)
        elif c == "3":
            dg = fb.DeviceGraph.generate_rmat(fb.RmatParams(24, 16, seed=3), relabel_bfs=True, **kw)
        elif c == "4":
            dg = fb.DeviceGraph.generate_chunglu(1 << 26, 1_200_000_000, seed=4, **kw)
        else:
            dg = fb.DeviceGraph.generate_rmat(fb.RmatParams(28, 16, seed=5), **kw)
        with dg:
            # unblocked reference run on the same handle (FUSED is never blocked; EC via a fresh handle is costly,
            # so compare against the lockstep-free plain EC of an unblocked handle in the same process below)
            res = {}
            for sh in shifts:
                os.environ["FPR_B200_BLOCK_SHIFT"] = str(sh)
                dg2 = dg  # blocked layout is built at the first EC run of the handle
                t0 = time.perf_counter()
                r = dg2.run(fb.ENGINE_EC, cfg, copy_ranks=False)
                t1 = time.perf_counter()
                r2 = dg2.run(fb.ENGINE_EC, cfg, copy_ranks=True)
                ms = r2.solve_ms / r2.trace.iterations
                res[sh] = r2.ranks.values
                print(f"cfg{c} reorder={int(reorder)} blocked shift={sh}: {r2.trace.iterations} it, {ms:.3f} ms/it, "
                      f"{dg.m / ms / 1e6:.1f} GTEPS, first run incl. build {1e3*(t1-t0):.0f} ms",
                      flush=True)
                break  # one layout per handle
        # unblocked
        if c == "2":
            dg = fb.DeviceGraph.generate_uniform(1 << 22, 16, 2, reorder=reorder)
        elif c == "3":
            dg = fb.DeviceGraph.generate_rmat(fb.RmatParams(24, 16, seed=3), relabel_bfs=True, reorder=reorder)
        elif c == "4":
            dg = fb.DeviceGraph.generate_chunglu(1 << 26, 1_200_000_000, seed=4, reorder=reorder)
        else:
            dg = fb.DeviceGraph.generate_rmat(fb.RmatParams(28, 16, seed=5), reorder=reorder)
        with dg:
            r = dg.run(fb.ENGINE_EC, cfg, copy_ranks=True)
            ms = r.solve_ms / r.trace.iterations
            d = np.max(np.abs(r.ranks.values - res[shifts[0]]) / r.ranks.values)
            print(f"cfg{c} reorder={int(reorder)} plain: {r.trace.iterations} it, {ms:.3f} ms/it, "
                  f"{dg.m / ms / 1e6:.1f} GTEPS; blocked vs plain max rel {d:.2e}", flush=True)
