"""EC/FusEd per-iteration time with and without FPR_B200_OPT_REORDER on configs 3-5 (natural/BFS/random order)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_2203_09284_b200 as fb
cfg = fb.PageRankConfig(threshold=1e-10)
which = sys.argv[1:] or ["3", "4", "5", "2"]
for c in which:
    for reorder in (False, True):
        if c == "3":
            dg = fb.DeviceGraph.generate_rmat(fb.RmatParams(24, 16, seed=3), relabel_bfs=True, reorder=reorder)
        elif c == "4":
            dg = fb.DeviceGraph.generate_chunglu(1 << 26, 1_200_000_000, seed=4, reorder=reorder)
        elif c == "5":
            dg = fb.DeviceGraph.generate_rmat(fb.RmatParams(28, 16, seed=5), reorder=reorder)
        else:
            dg = fb.DeviceGraph.generate_uniform(1 << 22, 16, 2, reorder=reorder)
        with dg:
            for eng, name in ((fb.ENGINE_EC, "ec"), (fb.ENGINE_FUSED, "fused")):
                r = dg.run(eng, cfg, copy_ranks=False)
                ms = r.solve_ms / r.trace.iterations
                print(f"config{c} reorder={int(reorder)} {name}: {r.trace.iterations} it, {ms:.3f} ms/it, "
                      f"{dg.m / ms / 1e6:.1f} GTEPS, converge {r.solve_ms:.1f} ms", flush=True)
