"""Bench-style step time (init + EC solve + status readback) for the library in FPR_B200_LIB."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2203_09284_b200 as fb
dg = fb.DeviceGraph.generate_uniform(1 << 22, 16, 2, stream=fb.torch_stream_handle())
cfg = fb.PageRankConfig(threshold=1e-10)
for _ in range(5):
    dg.run(fb.ENGINE_EC, cfg, copy_ranks=False, copy_trace=False)
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
torch.cuda.synchronize(); e0.record()
ks = []
for _ in range(50):
    r = dg.run(fb.ENGINE_EC, cfg, copy_ranks=False, copy_trace=False); ks.append(r.solve_ms)
e1.record(); torch.cuda.synchronize()
ms = e0.elapsed_time(e1) / 50
print(f"{os.environ.get('FPR_B200_LIB','base').split('_')[-1]}: step {ms:.4f} ms, kernel {sum(ks)/len(ks):.4f} ms, "
      f"value {dg.m * r.trace.iterations / ms / 1e6:.1f} GTEPS")
