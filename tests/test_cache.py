"""FPRG cache interop (graph_cache.hpp): files written here load in the
reference and vice versa, byte for byte; error behaviour mirrors
io_ingest_test.cpp:171-244 (truncation, bad magic, bad version)."""
import ctypes as C
import os

import numpy as np
import pytest

from oracle import REF_SO
from paper_2203_09284_b200 import Graph
from paper_2203_09284_b200.cache import CacheError, load_cache, save_cache


def _graph(oracle):
    n, s, d = oracle.generate_rmat(10, 16, seed=42)
    g = oracle.build_csr(n, s, d)
    return Graph(g.n, g.m, g.in_start, g.in_src, g.out_degree)


def test_roundtrip(oracle, tmp_path):
    g = _graph(oracle)
    p = str(tmp_path / "g.fprg")
    save_cache(g, p)
    h = load_cache(p)
    assert h.n == g.n and h.m == g.m
    for k in ("in_start", "in_src", "out_degree"):
        np.testing.assert_array_equal(getattr(h, k), getattr(g, k))
    assert os.path.getsize(p) == 4 + 4 + 16 + 8 * (2 * g.n + 1 + g.m)


@pytest.mark.skipif(not os.path.exists(REF_SO), reason="reference shim not built")
def test_interop_with_reference(oracle, tmp_path):
    L = C.CDLL(REF_SO)
    g = _graph(oracle)
    mine, theirs = str(tmp_path / "mine.fprg"), str(tmp_path / "ref.fprg")
    save_cache(g, mine)
    u64 = np.ctypeslib.ndpointer(np.uint64, flags="C_CONTIGUOUS")
    L.ref_save_cache.argtypes = [C.c_uint64, C.c_uint64, u64, u64, u64, C.c_char_p]
    assert L.ref_save_cache(g.n, g.m, g.in_start, g.in_src, g.out_degree, theirs.encode()) == 0
    assert open(mine, "rb").read() == open(theirs, "rb").read()
    L.ref_load_cache.argtypes = [C.c_char_p, C.POINTER(C.c_uint64), C.POINTER(C.c_uint64),
                                 C.c_void_p, C.c_void_p, C.c_void_p]
    n, m = C.c_uint64(), C.c_uint64()
    assert L.ref_load_cache(mine.encode(), C.byref(n), C.byref(m), None, None, None) == 0
    assert (n.value, m.value) == (g.n, g.m)


def test_errors(oracle, tmp_path):
    g = _graph(oracle)
    p = str(tmp_path / "g.fprg")
    save_cache(g, p)
    data = open(p, "rb").read()
    with pytest.raises(CacheError, match="cannot open"):
        load_cache(str(tmp_path / "missing.fprg"))
    open(p, "wb").write(data[:100])
    with pytest.raises(CacheError, match="truncated"):
        load_cache(p)
    open(p, "wb").write(b"XPRG" + data[4:])
    with pytest.raises(CacheError, match="bad magic"):
        load_cache(p)
    open(p, "wb").write(data[:4] + np.uint32(2).tobytes() + data[8:])
    with pytest.raises(CacheError, match="unsupported format version 2"):
        load_cache(p)
