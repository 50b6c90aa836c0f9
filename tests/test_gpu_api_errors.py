"""C-ABI error behaviour beyond the reference's validation messages: every
entry point rejects misuse with a status (never a crash), and leaves the
handle usable afterwards."""
import ctypes as C

import numpy as np
import pytest

import paper_2203_09284_b200 as fb
from paper_2203_09284_b200.dist import B200Part

pytestmark = pytest.mark.gpu


def _small():
    n, s, d = 5, np.array([0, 1, 2, 3, 4, 0], np.uint64), np.array([1, 2, 3, 4, 0, 2], np.uint64)
    return fb.build_csr(n, s, d)


def test_run_errors_cap_too_small():
    g = _small()
    L = fb.lib()
    with fb.DeviceGraph.from_graph(g) as dg:
        cfg = fb.PageRankConfig(threshold=1e-15)._c()
        errs = np.empty(2, np.float64)
        res = fb._Result()
        rc = L.fpr_b200_run(dg._h, fb.ENGINE_EC, C.byref(cfg), None, errs.ctypes.data, None, None, 2, C.byref(res))
        assert rc == fb.EINVAL and b"errors buffer" in L.fpr_b200_last_error()
        r = dg.run(fb.ENGINE_EC, fb.PageRankConfig(threshold=1e-10))  # still usable
        assert r.trace.converged


def test_unknown_engine_and_null_handles():
    L = fb.lib()
    cfg = fb.PageRankConfig()._c()
    res = fb._Result()
    assert L.fpr_b200_run(None, 0, C.byref(cfg), None, None, None, None, 0, C.byref(res)) == fb.EINVAL
    with fb.DeviceGraph.from_graph(_small()) as dg:
        with pytest.raises(ValueError, match="unknown engine"):
            dg.run(7, fb.PageRankConfig())
    assert L.fpr_b200_graph_set_wave_count(None, 2) == fb.EINVAL
    assert L.fpr_b200_part_init(None, None) == fb.EINVAL
    assert L.fpr_b200_ipc_close(C.c_void_p(0x1234)) == fb.EINVAL


def test_part_misuse():
    L = fb.lib()
    with fb.DeviceGraph.from_graph(_small()) as full:
        part = B200Part(full, 2, 0)
    cfg = fb.PageRankConfig()._c()
    buf = __import__("torch").zeros(2 * part.slice, dtype=__import__("torch").float64, device="cuda")
    pair = __import__("torch").zeros(2, dtype=__import__("torch").float64, device="cuda")
    rc = L.fpr_b200_part_sweep(part.graph._h, fb.ENGINE_EC, C.byref(cfg), buf.data_ptr(), buf.data_ptr(),
                               pair.data_ptr())
    assert rc == fb.EINVAL and b"part_init" in L.fpr_b200_last_error()
    out = np.empty(part.n_local, np.float64)
    assert L.fpr_b200_part_ranks_prev(part.graph._h, out.ctypes.data) == fb.EINVAL
    part.init(buf)
    rc = L.fpr_b200_part_sweep_peers(part.graph._h, fb.ENGINE_EC, C.byref(cfg), buf.data_ptr(), buf.data_ptr(),
                                     None, 3, pair.data_ptr())
    assert rc == fb.EINVAL  # peer count must equal nparts
    with pytest.raises(ValueError, match="nparts"):
        with fb.DeviceGraph.from_graph(_small()) as full:
            B200Part(full, 0, 0)
    part.close()


def test_parse_cap_too_small_reports_m():
    L = fb.lib()
    text = b"1 2\n2 3\n3 1\n"
    n, m = C.c_uint64(), C.c_uint64()
    edges = np.empty(2, np.uint64)
    err = fb._ParseErr()
    rc = L.fpr_b200_parse_edge_list(text, len(text), None, C.byref(n), C.byref(m), edges.ctypes.data, 1,
                                    C.byref(err))
    assert rc == fb.ERANGE and (n.value, m.value) == (3, 3)


def test_from_edges_length_mismatch_and_range():
    with pytest.raises(ValueError, match="lengths differ"):
        fb.DeviceGraph.from_edges(3, [0, 1], [1])
    with pytest.raises(ValueError, match="n >= 2"):
        fb.DeviceGraph.from_edges(1 << 31, [0], [1])


def test_gate_misuse():
    """Device-side stop rule (fpr_b200_gate_*, fpr_b200_part_ranks_after):
    null gates, pair counts outside 1..8 and sweeps beyond those issued are
    EINVAL; a gate reads back 0 iterations after init."""
    import torch

    L = fb.lib()
    cfg = fb.PageRankConfig()._c()
    assert L.fpr_b200_gate_init(None, 4, 0, None) == fb.EINVAL
    gate = torch.zeros(int(L.fpr_b200_gate_bytes(4)), dtype=torch.uint8, device="cuda")
    assert L.fpr_b200_gate_init(gate.data_ptr(), 4, 0, None) == fb.OK
    pairs = torch.zeros(18, dtype=torch.float64, device="cuda")
    arr = (C.c_void_p * 9)(*[pairs.data_ptr() + 16 * r for r in range(9)])
    assert L.fpr_b200_gate_update(gate.data_ptr(), arr, 0, C.byref(cfg), 0, 0, None) == fb.EINVAL
    assert L.fpr_b200_gate_update(gate.data_ptr(), arr, 9, C.byref(cfg), 0, 0, None) == fb.EINVAL
    it, st = C.c_uint64(7), C.c_int(7)
    assert L.fpr_b200_gate_read(gate.data_ptr(), 0, None, C.byref(it), C.byref(st), None, None, 0) == fb.OK
    assert it.value == 0 and st.value == 0
    # one update with a zero residual: the rule holds, the gate stops and stays stopped
    assert L.fpr_b200_gate_update(gate.data_ptr(), arr, 2, C.byref(cfg), 0, 0, None) == fb.OK
    assert L.fpr_b200_gate_update(gate.data_ptr(), arr, 2, C.byref(cfg), 0, 0, None) == fb.OK
    assert L.fpr_b200_gate_read(gate.data_ptr(), 0, None, C.byref(it), C.byref(st), None, None, 0) == fb.OK
    assert it.value == 1 and st.value == 1
    with fb.DeviceGraph.from_graph(_small()) as full:
        part = B200Part(full, 1, 0)
        out = np.empty(part.n_local)
        assert L.fpr_b200_part_ranks_after(part.graph._h, 0, out.ctypes.data) == fb.EINVAL  # before part_init
        ex = torch.zeros(part.slice, dtype=torch.float64, device="cuda")
        part.init(ex)
        assert L.fpr_b200_part_ranks_after(part.graph._h, 1, out.ctypes.data) == fb.EINVAL  # none issued
        assert L.fpr_b200_part_ranks_after(part.graph._h, 0, out.ctypes.data) == fb.OK
        assert np.allclose(out, 1.0 / 5)
        part.close()
