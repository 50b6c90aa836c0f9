"""EC / FusEd / lockstep on configs 3-5 with no reorder, FPR_B200_OPT_REORDER_SOURCES
("sources") and FPR_B200_OPT_REORDER ("degree"): python scripts/reorder_sources_probe.py [configs]"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2203_09284_b200 as fb
from pb_probe import make

cfg = fb.PageRankConfig(threshold=1e-10)
for c in (sys.argv[1:] or ["3", "4", "5"]):
    for ro in (False, "sources", "degree"):
        with make(c, reorder=ro) as dg:
            out = []
            for eng, tag in ((fb.ENGINE_EC, "ec"), (fb.ENGINE_FUSED, "fused"), (fb.ENGINE_FUSED_LOCKSTEP, "lockstep")):
                r = dg.run(eng, cfg, copy_ranks=False)
                out.append(f"{tag} {r.trace.iterations} it x {r.solve_ms / r.trace.iterations:.3f} = {r.solve_ms:.1f} ms")
            print(f"cfg{c} reorder={ro}: " + "; ".join(out), flush=True)
