"""One resident-graph solve for profiling: python scripts/profile_solve.py [engine] [config] [reps]
engine: ec | fused | lockstep ; config: 1 (R-MAT s16) | 2 (uniform 2^22) | 3 (R-MAT s24, no relabel)
| 3b (config 3: R-MAT s24 + BFS relabel); env MAXIT caps the iterations per solve"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2203_09284_b200 as fb

eng = {"ec": fb.ENGINE_EC, "fused": fb.ENGINE_FUSED, "lockstep": fb.ENGINE_FUSED_LOCKSTEP}[sys.argv[1] if len(sys.argv) > 1 else "ec"]
cfgn = sys.argv[2] if len(sys.argv) > 2 else "2"
reps = int(sys.argv[3]) if len(sys.argv) > 3 else 2
if cfgn == "1":
    dg = fb.DeviceGraph.generate_rmat(fb.RmatParams(16, 16, seed=1))
elif cfgn == "3b":
    dg = fb.DeviceGraph.generate_rmat(fb.RmatParams(24, 16, seed=3), relabel_bfs=True)
elif cfgn == "3":
    dg = fb.DeviceGraph.generate_rmat(fb.RmatParams(24, 16, seed=3))
else:
    dg = fb.DeviceGraph.generate_uniform(1 << 22, 16, 2)
cfg = fb.PageRankConfig(threshold=1e-10, max_iterations=int(os.environ.get("MAXIT", "10000")))
for _ in range(reps):
    r = dg.run(eng, cfg, copy_ranks=False)
    print(f"n={dg.n} m={dg.m} iters={r.trace.iterations} solve_ms={r.solve_ms:.3f} "
          f"GTEPS={dg.m * r.trace.iterations / r.solve_ms / 1e6:.1f} "
          f"iter_us={[round(x / 1e3, 1) for x in r.trace.iter_ns]}")
