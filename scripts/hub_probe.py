"""EC ms/sweep with FPR_B200_OPT_REORDER at several FPR_B200_HUB_MIN thresholds: python scripts/hub_probe.py 3 4 5"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2203_09284_b200 as fb
cfg = fb.PageRankConfig(threshold=1e-10)
for c in sys.argv[1:]:
    for hm in (os.environ.get("HUBS", "0,16,64,256,1024").split(",")):
        os.environ["FPR_B200_HUB_MIN"] = hm
        if c == "3":
            dg = fb.DeviceGraph.generate_rmat(fb.RmatParams(24, 16, seed=3), relabel_bfs=True, reorder=True)
        elif c == "4":
            dg = fb.DeviceGraph.generate_chunglu(1 << 26, 1_200_000_000, seed=4, reorder=True)
        else:
            dg = fb.DeviceGraph.generate_rmat(fb.RmatParams(28, 16, seed=5), reorder=True)
        with dg:
            r = dg.run(fb.ENGINE_EC, cfg, copy_ranks=False)
            f = dg.run(fb.ENGINE_FUSED, cfg, copy_ranks=False)
            print(f"cfg{c} hub_min={hm}: ec {r.solve_ms / r.trace.iterations:.3f} ms/it; fused {f.trace.iterations} it "
                  f"{f.solve_ms:.1f} ms", flush=True)
