"""Propagation-blocked lockstep (FusEd schedule on PB sweeps) vs PB EC, plain
lockstep and async FusEd: python scripts/pb_lockstep_probe.py [configs]
(env WAVES="4,8,16,32")."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2203_09284_b200 as fb
from pb_probe import make  # noqa: E402  (graph factories by config name)

cfg = fb.PageRankConfig(threshold=1e-10)
waves = [int(x) for x in os.environ.get("WAVES", "4,8,16,32").split(",")]


def show(tag, c, dg, r):
    ms = r.solve_ms / r.trace.iterations
    print(f"cfg{c} {tag}: {r.trace.iterations} it, {ms:.3f} ms/sweep, {r.solve_ms:.1f} ms to converge, "
          f"{dg.m / ms / 1e6:.1f} GTEPS", flush=True)


for c in (sys.argv[1:] or ["4", "5"]):
    with make(c, reorder=c.endswith("r"), pb=True) as dg:
        show("pb ec", c, dg, dg.run(fb.ENGINE_EC, cfg, copy_ranks=False))
        for w in waves:
            dg.set_wave_count(w)
            show(f"pb lockstep {w:2d} waves", c, dg, dg.run(fb.ENGINE_FUSED_LOCKSTEP, cfg, copy_ranks=False))
        show("async fused (plain sweeps)", c, dg, dg.run(fb.ENGINE_FUSED, cfg, copy_ranks=False))
