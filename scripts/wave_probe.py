"""Lockstep sweeps and time vs wave count: python scripts/wave_probe.py [config]"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2203_09284_b200 as fb
c = sys.argv[1] if len(sys.argv) > 1 else "2"
cfg = fb.PageRankConfig(threshold=1e-10)
waves = [int(x) for x in sys.argv[2].split(",")] if len(sys.argv) > 2 else [1, 2, 3, 4, 5, 8, 16, 32]
if c == "2":
    dg = fb.DeviceGraph.generate_uniform(1 << 22, 16, 2)
elif c == "3":
    dg = fb.DeviceGraph.generate_rmat(fb.RmatParams(24, 16, seed=3), relabel_bfs=True)
elif c == "4":
    dg = fb.DeviceGraph.generate_chunglu(1 << 26, 1_200_000_000, seed=4)
else:
    dg = fb.DeviceGraph.generate_rmat(fb.RmatParams(28, 16, seed=5), reorder=c.endswith("r"))
with dg:
    for w in waves:
        dg.set_wave_count(w)
        r = dg.run(fb.ENGINE_FUSED_LOCKSTEP, cfg, copy_ranks=False)
        print(f"cfg{c} waves={w}: {r.trace.iterations} sweeps, {r.solve_ms / r.trace.iterations * 1e3:.0f} us/sweep, "
              f"{r.solve_ms:.2f} ms", flush=True)
