"""Config-2 edges rendered as fixed-width decimal text (shared by the ingest probes and bench.py)."""
import numpy as np


def render_fixed(src, dst, width=7):
    """"%0{width}d %0{width}d\\n" per edge (leading zeros are valid tokens, edge_list.hpp:25-30)."""
    e = len(src)
    out = np.empty((e, 2 * width + 2), np.uint8)
    for col, ids in ((0, src), (width + 1, dst)):
        v = np.asarray(ids, dtype=np.uint64).copy()
        for k in range(width - 1, -1, -1):
            out[:, col + k] = (v % np.uint64(10)).astype(np.uint8) + 48
            v //= np.uint64(10)
    out[:, width] = 32
    out[:, 2 * width + 1] = 10
    return out.reshape(-1)


def config2_text():
    import paper_2203_09284_b200 as fb

    dg = fb.DeviceGraph.generate_uniform(1 << 22, 16, 2)
    g = dg.download()
    dg.close()
    dst = np.repeat(np.arange(g.n, dtype=np.uint64), np.diff(g.in_start.astype(np.int64)))
    return render_fixed(g.in_src, dst)
