"""Source-blocked EC on config 3 at block sizes 2^21-2^23, natural and sources-first order."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.abspath(__file__))); sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2203_09284_b200 as fb
from pb_probe import make
cfg = fb.PageRankConfig(threshold=1e-10)
for sh in (21, 22, 23):
    os.environ["FPR_B200_BLOCK_SHIFT"] = str(sh)
    for ro in (False, "sources"):
        with make("3", reorder=ro, blocked=True) as dg:
            dg.run(fb.ENGINE_EC, fb.PageRankConfig(threshold=1e-10, max_iterations=1), copy_ranks=False)
            r = dg.run(fb.ENGINE_EC, cfg, copy_ranks=False)
            print(f"cfg3 blocked 2^{sh} reorder={ro}: {r.trace.iterations} it x {r.solve_ms / r.trace.iterations:.3f} ms", flush=True)
