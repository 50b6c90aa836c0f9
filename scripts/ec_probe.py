"""EC ms/sweep on configs for the library in FPR_B200_LIB: python scripts/ec_probe.py 4 5r"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2203_09284_b200 as fb
cfg = fb.PageRankConfig(threshold=1e-10)
tag = os.environ.get("FPR_B200_LIB", "base").split("_")[-1]
for c in sys.argv[1:]:
    if c == "2":
        dg = fb.DeviceGraph.generate_uniform(1 << 22, 16, 2)
    elif c == "3":
        dg = fb.DeviceGraph.generate_rmat(fb.RmatParams(24, 16, seed=3), relabel_bfs=True)
    elif c == "4":
        dg = fb.DeviceGraph.generate_chunglu(1 << 26, 1_200_000_000, seed=4)
    else:
        dg = fb.DeviceGraph.generate_rmat(fb.RmatParams(28, 16, seed=5), reorder=c.endswith("r"))
    with dg:
        r = dg.run(fb.ENGINE_EC, cfg, copy_ranks=False)
        print(f"{tag} cfg{c} ec: {r.trace.iterations} it, {r.solve_ms / r.trace.iterations:.3f} ms/it", flush=True)
