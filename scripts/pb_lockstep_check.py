"""PB lockstep vs its CPU restatement on R-MAT with the BFS relabel (config 3's
shape at small scale): python scripts/pb_lockstep_check.py [scale]"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_2203_09284_b200 as fb
from oracle import Oracle

sc = int(sys.argv[1]) if len(sys.argv) > 1 else 16
o = Oracle()
with fb.DeviceGraph.generate_rmat(fb.RmatParams(sc, 16, seed=3), relabel_bfs=True) as dg:
    g = dg.download()
og = o.build_csr(g.n, g.in_src, np.repeat(np.arange(g.n, dtype=np.uint64), np.diff(g.in_start.astype(np.int64))))
cfg = fb.PageRankConfig(threshold=1e-10)
ec = o.pagerank_ec(og, threshold=1e-10)
for waves in (4, 8, 32):
    with fb.DeviceGraph.from_graph(g, pb=True, wave_count=waves) as d:
        ws = d.wave_starts(waves)
        ref = o.pagerank_lockstep(og, ws, threshold=1e-10)
        r = d.run(fb.ENGINE_FUSED_LOCKSTEP, cfg)
    with fb.DeviceGraph.from_graph(g, wave_count=waves) as d:
        ws2 = d.wave_starts(waves)
        ref2 = o.pagerank_lockstep(og, ws2, threshold=1e-10)
        r2 = d.run(fb.ENGINE_FUSED_LOCKSTEP, cfg)
    print(f"s{sc} waves={waves}: EC {ec.iterations}; PB lockstep gpu {r.trace.iterations} oracle {ref.iterations} "
          f"(starts {list(ws[:4])}...); pull lockstep gpu {r2.trace.iterations} oracle {ref2.iterations} "
          f"(starts {list(ws2[:4])}...)", flush=True)
