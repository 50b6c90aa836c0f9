"""Per-iteration floor: run to threshold 1e-300 (until the fp64 fixed point) on
small uniform graphs; iter_ns gives the grid-barrier + single-task latency floor."""
import os, sys
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2203_09284_b200 as fb
for n, deg in ((64, 2), (4096, 4), (65536, 16), (1 << 20, 16)):
    with fb.DeviceGraph.generate_uniform(n, deg, 7) as dg:
        for eng, name in ((fb.ENGINE_EC, "ec"), (fb.ENGINE_FUSED, "fused"), (fb.ENGINE_FUSED_LOCKSTEP, "lockstep")):
            r = dg.run(eng, fb.PageRankConfig(threshold=1e-300, max_iterations=100))
            ns = r.trace.iter_ns[1:].astype(float)
            print(f"n={n} m={dg.m} tasks={dg.ntasks} {name}: iters {r.trace.iterations} median iter {np.median(ns)/1e3:.2f} us, min {ns.min()/1e3:.2f} us, solve {r.solve_ms:.3f} ms")
