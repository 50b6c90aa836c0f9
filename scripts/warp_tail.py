"""Per-warp finish times within EC sweep 3.  Needs the diagnostic build:
make -C paper_2203_09284_b200/csrc variant V=trace EXTRA=-DFPR_TRACE_WARPS, then
FPR_B200_LIB=paper_2203_09284_b200/csrc/build/libfpr_b200_trace.so python scripts/warp_tail.py"""
import ctypes as C, os, sys
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2203_09284_b200 as fb
dg = fb.DeviceGraph.generate_uniform(1 << 22, 16, 2)
r = dg.run(fb.ENGINE_EC, fb.PageRankConfig(threshold=1e-10), copy_ranks=False)
nw = 592 * 5
out = np.zeros(nw + 5, np.uint64)
fb.lib().fpr_b200_debug_warp_times(dg._h, out.ctypes.data, C.c_uint64(nw))
w = out[:nw].astype(np.float64)
ns = out[nw:].astype(np.float64)
t0 = ns[2]
rel = (w - t0) / 1e3
print(f"sweep 3: start->end {(ns[3]-ns[2])/1e3:.1f} us; warp finish: min {rel.min():.1f} p10 {np.percentile(rel,10):.1f} "
      f"median {np.median(rel):.1f} p90 {np.percentile(rel,90):.1f} max {rel.max():.1f} us")
