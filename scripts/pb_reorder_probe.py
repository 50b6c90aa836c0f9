"""PB EC / lockstep with and without the sources-first reorder: python scripts/pb_reorder_probe.py"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.abspath(__file__))); sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2203_09284_b200 as fb
from pb_probe import make
cfg = fb.PageRankConfig(threshold=1e-10)
for c in ["4", "5"]:
    for ro in (False, "sources"):
        with make(c, reorder=ro, pb=True) as dg:
            out = []
            for eng, tag in ((fb.ENGINE_EC, "pb ec"), (fb.ENGINE_FUSED_LOCKSTEP, "pb lockstep")):
                dg.run(eng, fb.PageRankConfig(threshold=1e-10, max_iterations=1), copy_ranks=False)
                r = dg.run(eng, cfg, copy_ranks=False)
                out.append(f"{tag} {r.trace.iterations} it x {r.solve_ms / r.trace.iterations:.3f} = {r.solve_ms:.1f} ms")
            print(f"cfg{c} reorder={ro}: " + "; ".join(out), flush=True)
