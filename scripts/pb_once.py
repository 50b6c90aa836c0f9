"""Two propagation-blocked EC sweeps on one config (for ncu): python scripts/pb_once.py 4"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2203_09284_b200 as fb

c = sys.argv[1] if len(sys.argv) > 1 else "4"
if c == "2":
    dg = fb.DeviceGraph.generate_uniform(1 << 22, 16, 2, pb=True)
elif c == "3":
    dg = fb.DeviceGraph.generate_rmat(fb.RmatParams(24, 16, seed=3), relabel_bfs=True, pb=True)
elif c == "4":
    dg = fb.DeviceGraph.generate_chunglu(1 << 26, 1_200_000_000, seed=4, pb=True)
else:
    dg = fb.DeviceGraph.generate_rmat(fb.RmatParams(28, 16, seed=5), pb=True)
with dg:
    r = dg.run(fb.ENGINE_EC, fb.PageRankConfig(threshold=1e-10, max_iterations=2), copy_ranks=False)
    print(f"cfg{c} pb: {r.solve_ms / 2:.3f} ms/sweep, m={dg.m}")
