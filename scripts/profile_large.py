"""One short EC launch (2 sweeps) on config 4 or 5 (optionally reordered) for ncu:
python scripts/profile_large.py 4|5|5r"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2203_09284_b200 as fb
c = sys.argv[1]
if c == "4":
    dg = fb.DeviceGraph.generate_chunglu(1 << 26, 1_200_000_000, seed=4)
else:
    dg = fb.DeviceGraph.generate_rmat(fb.RmatParams(28, 16, seed=5), reorder=c.endswith("r"))
with dg:
    r = dg.run(fb.ENGINE_EC, fb.PageRankConfig(threshold=1e-10, max_iterations=2), copy_ranks=False)
    print(f"cfg{c}: n={dg.n} m={dg.m} 2 sweeps {r.solve_ms:.2f} ms")
