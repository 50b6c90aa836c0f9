"""Edge-list ingest throughput: config-2 edges rendered as fixed-width decimal
text ("%07d %07d\\n"), then text -> device CSR (fpr_b200_graph_from_edge_list)
and text -> EdgeSet (parse only), vs the reference parse_edge_list+build_csr
on a sample."""
import os, sys, time
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2203_09284_b200 as fb


def render_fixed(src, dst, width=7):
    e = len(src)
    out = np.empty((e, 2 * width + 2), np.uint8)
    for col, ids in ((0, src), (width + 1, dst)):
        v = ids.astype(np.uint64).copy()
        for k in range(width - 1, -1, -1):
            out[:, col + k] = (v % 10).astype(np.uint8) + 48
            v //= 10
    out[:, width] = 32
    out[:, 2 * width + 1] = 10
    return out.reshape(-1)


dg = fb.DeviceGraph.generate_uniform(1 << 22, 16, 2)
g = dg.download(); dg.close()
dst = np.repeat(np.arange(g.n, dtype=np.uint64), np.diff(g.in_start.astype(np.int64)))
t0 = time.perf_counter(); text = render_fixed(g.in_src, dst); t1 = time.perf_counter()
print(f"rendered {len(text)/1e9:.2f} GB ({g.m} edges) in {t1-t0:.1f} s", flush=True)
pinned = torch.empty(len(text), dtype=torch.uint8, pin_memory=True); pinned.numpy()[:] = text
for label, buf in (("pageable", text), ("pinned", pinned.numpy())):
    for rep in range(3):
        torch.cuda.synchronize(); t0 = time.perf_counter()
        d = fb.DeviceGraph.from_edge_list(buf)
        torch.cuda.synchronize(); t1 = time.perf_counter()
        m = d.m; d.close()
        print(f"{label} text->CSR: {1e3*(t1-t0):.1f} ms, {len(text)/(t1-t0)/1e9:.2f} GB/s, "
              f"{g.m/(t1-t0)/1e6:.0f} M edges/s (m={m})", flush=True)
t0 = time.perf_counter(); es = fb.parse_edge_list(pinned.numpy()); t1 = time.perf_counter()
print(f"pinned parse -> host EdgeSet: {1e3*(t1-t0):.1f} ms (n={es.n})", flush=True)
assert m == g.m
# the reference on a 1/32 sample (CPU, single thread: parse_edge_list is sequential)
try:
    from oracle import load_reference
    ref = load_reference()
    sample = text[: (len(text) // 32 // 16) * 16].tobytes()
    t0 = time.perf_counter(); p = ref.parse_edge_list(sample); t1 = time.perf_counter()
    t2 = time.perf_counter(); ref.build_csr(p.n, p.edges[:, 0], p.edges[:, 1]); t3 = time.perf_counter()
    e = len(p.edges)
    print(f"reference sample {len(sample)/1e6:.0f} MB ({e} edges): parse {t1-t0:.2f} s "
          f"({e/(t1-t0)/1e6:.2f} M edges/s), build_csr {t3-t2:.2f} s", flush=True)
except Exception as ex:  # noqa
    print("reference unavailable:", ex)
