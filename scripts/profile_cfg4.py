import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2203_09284_b200 as fb
reorder = len(sys.argv) > 1 and sys.argv[1] == "1"
with fb.DeviceGraph.generate_chunglu(1 << 26, 1_200_000_000, seed=4, reorder=reorder) as dg:
    r = dg.run(fb.ENGINE_EC, fb.PageRankConfig(threshold=1e-10, max_iterations=3), copy_ranks=False)
    print("iters", r.trace.iterations, "ms", r.solve_ms)
