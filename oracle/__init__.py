"""CPU checkers for the FusEd-PageRank hot path -- TEST INFRASTRUCTURE ONLY.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s cpu-baseline /
``--impl reference`` legs import this package.  The product
(``paper_2203_09284_b200``) never does; it has no CPU fallback.

Two checkers, both loaded with ctypes:

* ``Oracle``    -- ``oracle/libfpr_oracle.so``, the C restatement
  (``oracle/fpr_oracle.c``), pinned against the reference by
  ``tests/test_oracle.py`` + ``tests/golden/``.
* ``Reference`` -- ``oracle/_ref/libfpr_ref.so``, the reference headers of
  ``/root/reference/proj/include`` compiled unmodified (``oracle/Makefile``).
  Present wherever it was built (it travels to the GPU box with the repo
  snapshot); ``load_reference()`` returns None when it is missing.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess
from dataclasses import dataclass

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ORACLE_SO = os.path.join(HERE, "libfpr_oracle.so")
REF_SO = os.path.join(HERE, "_ref", "libfpr_ref.so")

NORM_LINF = 0
NORM_L1 = 1

_u64p = np.ctypeslib.ndpointer(dtype=np.uint64, flags="C_CONTIGUOUS")
_f64p = np.ctypeslib.ndpointer(dtype=np.float64, flags="C_CONTIGUOUS")
_u64 = C.c_uint64
_f64 = C.c_double


@dataclass
class Graph:
    """Mirror of ``fpr::Graph`` (graph.hpp:20-30): dst-grouped in-CSR, u64."""

    n: int
    m: int
    in_start: np.ndarray  # u64[n+1]
    in_src: np.ndarray  # u64[m]
    out_degree: np.ndarray  # u64[n]

    def in_degree(self) -> np.ndarray:
        return np.diff(self.in_start)


@dataclass
class Run:
    ranks: np.ndarray
    errors: np.ndarray
    l1_errors: np.ndarray | None
    iterations: int
    history: np.ndarray | None = None
    seconds: float = 0.0

    @property
    def converged_linf(self) -> bool:  # unused helper for readability in tests
        return True


@dataclass
class Parsed:
    """``fpr::EdgeSet`` from ``parse_edge_list`` (edge_list.hpp:39-80), or the
    ``ParseError`` it threw (error_line > 0, error = what())."""

    n: int
    edges: np.ndarray  # (m, 2) u64 dense ids, input order
    error_line: int = 0
    error: str = ""


_PARSE_WHAT = {1: "expected two integer tokens", 3: "trailing characters after edge"}


def _ensure_built() -> None:
    if not os.path.exists(ORACLE_SO):
        subprocess.run(["make", "-s", "-C", HERE, os.path.abspath(ORACLE_SO)], check=True)


class Oracle:
    """ctypes binding of the C restatement (fpr_oracle.h)."""

    def __init__(self) -> None:
        _ensure_built()
        L = C.CDLL(ORACLE_SO)
        L.fo_generate_rmat.argtypes = [C.c_uint32, _u64, _f64, _f64, _f64, _f64, _u64, _u64p, _u64p]
        L.fo_generate_rmat.restype = C.c_int
        L.fo_random_sparse.argtypes = [_u64, _u64, _u64, _u64p, _u64p]
        L.fo_random_sparse.restype = _u64
        L.fo_build_csr.argtypes = [_u64, _u64, _u64p, _u64p, _u64p, _u64p, _u64p,
                                   C.POINTER(_u64), C.POINTER(_u64)]
        L.fo_build_csr.restype = C.c_int
        eng = [_u64, _u64, _u64p, _u64p, _u64p, _f64, _f64, _u64, C.c_int]
        outs = [_f64p, _f64p, C.c_void_p, C.POINTER(_u64), C.c_void_p, _u64]
        L.fo_pagerank_ec.argtypes = eng + outs
        L.fo_pagerank_fused_seq.argtypes = eng + outs
        L.fo_pagerank_lockstep.argtypes = eng + [_u64, _u64p] + outs
        for f in (L.fo_pagerank_ec, L.fo_pagerank_fused_seq, L.fo_pagerank_lockstep):
            f.restype = C.c_int
        L.fo_dense_oracle.argtypes = [_u64, _u64p, _u64p, _u64p, _f64, _f64, _u64, _f64p]
        L.fo_dense_oracle.restype = C.c_int
        L.fo_bfs_relabel.argtypes = [_u64, _u64, _u64p, _u64p, _u64, _u64p]
        L.fo_bfs_relabel.restype = C.c_int
        L.fo_chunglu_cdf.argtypes = [_f64, _u64, _f64p]
        L.fo_chunglu_cdf.restype = None
        L.fo_chunglu_weight.argtypes = [_f64p, _u64, _u64, _u64]
        L.fo_chunglu_weight.restype = _u64
        L.fo_generate_chunglu.argtypes = [_u64, _u64, _f64, _u64, _u64, _u64p, _u64p]
        L.fo_generate_chunglu.restype = C.c_int
        L.fo_parse_edge_list.argtypes = [C.c_char_p, _u64, C.POINTER(_u64), C.POINTER(_u64), C.c_void_p,
                                         _u64, C.POINTER(_u64), C.POINTER(C.c_int), C.POINTER(_u64),
                                         C.POINTER(_u64)]
        L.fo_parse_edge_list.restype = C.c_int
        L.fo_ec_step.argtypes = [_u64, _u64p, _u64p, _u64p, _f64, _f64p, _f64p, C.POINTER(_f64), C.POINTER(_f64)]
        L.fo_ec_step.restype = C.c_int
        L.fo_l1_norm.argtypes = [_u64, _f64p, _f64p]
        L.fo_l1_norm.restype = _f64
        L.fo_linf_norm.argtypes = [_u64, _f64p, _f64p]
        L.fo_linf_norm.restype = _f64
        self.lib = L

    # ---- inputs -----------------------------------------------------------
    def generate_rmat(self, scale, edge_factor, a=0.57, b=0.19, c=0.19, d=0.05, seed=0):
        draws = edge_factor << scale
        src = np.empty(draws, np.uint64)
        dst = np.empty(draws, np.uint64)
        rc = self.lib.fo_generate_rmat(scale, edge_factor, a, b, c, d, seed, src, dst)
        if rc:
            raise ValueError("rmat: invalid parameters")
        return 1 << scale, src, dst

    def random_sparse(self, n, avg_degree, seed):
        src = np.empty(n * avg_degree, np.uint64)
        dst = np.empty(n * avg_degree, np.uint64)
        k = self.lib.fo_random_sparse(n, avg_degree, seed, src, dst)
        return n, src[:k].copy(), dst[:k].copy()

    def parse_edge_list(self, text: bytes) -> Parsed:
        """fo_parse_edge_list; the message restates ParseError::what()
        (edge_list.hpp:17-21, 60-73)."""
        n, m, line, tok_off, tok_len = _u64(0), _u64(0), _u64(0), _u64(0), _u64(0)
        kind = C.c_int(0)
        args = (C.byref(line), C.byref(kind), C.byref(tok_off), C.byref(tok_len))
        rc = self.lib.fo_parse_edge_list(text, len(text), C.byref(n), C.byref(m), None, 0, *args)
        if rc == 6:
            what = (_PARSE_WHAT[kind.value] if kind.value != 2 else
                    "bad token '" + text[tok_off.value:tok_off.value + tok_len.value].decode("latin-1") + "'")
            what = f"line {line.value}: {what}".split("\x00")[0]  # what() is a C string
            return Parsed(0, np.zeros((0, 2), np.uint64), line.value, what)
        if rc:
            raise MemoryError("fo_parse_edge_list")
        edges = np.empty((max(m.value, 1), 2), np.uint64)
        rc = self.lib.fo_parse_edge_list(text, len(text), C.byref(n), C.byref(m), edges.ctypes.data,
                                         m.value, *args)
        assert rc == 0
        return Parsed(n.value, edges[: m.value].copy())

    def build_csr(self, n, src, dst) -> Graph:
        src = np.ascontiguousarray(src, np.uint64)
        dst = np.ascontiguousarray(dst, np.uint64)
        in_start = np.empty(n + 1, np.uint64)
        in_src = np.empty(max(len(src), 1), np.uint64)
        out_degree = np.empty(max(n, 1), np.uint64)
        m = _u64(0)
        bad = _u64(0)
        rc = self.lib.fo_build_csr(n, len(src), src, dst, in_start, in_src, out_degree,
                                   C.byref(m), C.byref(bad))
        if rc == 1:
            i = bad.value
            raise ValueError(f"build_csr: edge #{i} ({src[i]},{dst[i]}) has endpoint outside [0,{n})")
        if rc:
            raise RuntimeError(f"fo_build_csr rc={rc}")
        return Graph(n, m.value, in_start, in_src[: m.value].copy(), out_degree[:n].copy())

    def bfs_relabel(self, g: Graph, root: int = 0) -> np.ndarray:
        """Config-3 crawl order: new_id[old]."""
        new_id = np.empty(g.n, np.uint64)
        in_src = g.in_src if g.m else np.zeros(1, np.uint64)
        if self.lib.fo_bfs_relabel(g.n, g.m, g.in_start, in_src, root, new_id):
            raise ValueError("bfs_relabel: invalid input")
        return new_id

    def relabel(self, g: Graph, new_id: np.ndarray) -> Graph:
        """build_csr of g's edges with ids mapped through new_id."""
        dst = np.repeat(np.arange(g.n, dtype=np.uint64), np.diff(g.in_start).astype(np.int64))
        return self.build_csr(g.n, new_id[g.in_src], new_id[dst])

    def chunglu_cdf(self, alpha: float, kmax: int) -> np.ndarray:
        cdf = np.empty(kmax, np.float64)
        self.lib.fo_chunglu_cdf(alpha, kmax, cdf)
        return cdf

    def generate_chunglu(self, n: int, draws: int, seed: int, alpha: float = 2.1, kmax: int = 1_000_000):
        src = np.empty(draws, np.uint64)
        dst = np.empty(draws, np.uint64)
        if self.lib.fo_generate_chunglu(n, draws, alpha, kmax, seed, src, dst):
            raise ValueError("chung-lu: invalid parameters")
        return n, src, dst

    # ---- engines ----------------------------------------------------------
    def _run(self, fn, g: Graph, damping, threshold, max_iterations, norm, extra, history_cap):
        ranks = np.empty(max(g.n, 1), np.float64)
        errors = np.empty(max_iterations, np.float64)
        l1 = np.empty(max_iterations, np.float64)
        it = _u64(0)
        hist = None
        hp = None
        if history_cap:
            hist = np.empty((history_cap, g.n), np.float64)
            hp = hist.ctypes.data
        in_src = g.in_src if g.m else np.zeros(1, np.uint64)
        rc = fn(g.n, g.m, g.in_start, in_src, g.out_degree, damping, threshold, max_iterations,
                norm, *extra, ranks, errors, l1.ctypes.data, C.byref(it), hp, history_cap)
        if rc:
            raise ValueError(f"pagerank: invalid configuration (rc={rc})")
        k = it.value
        return Run(ranks[: g.n], errors[:k].copy(), l1[:k].copy(), k,
                   None if hist is None else hist[: min(k, history_cap)])

    def pagerank_ec(self, g, damping=0.85, threshold=1e-15, max_iterations=10000,
                    norm=NORM_LINF, history_cap=0) -> Run:
        return self._run(self.lib.fo_pagerank_ec, g, damping, threshold, max_iterations, norm,
                         (), history_cap)

    def ec_step(self, g: Graph, prev: np.ndarray, damping=0.85):
        """One EC iteration from `prev` (OpenMP over rows; bit-identical to the
        sequential iteration).  Returns (next, max |delta|, sum |delta|)."""
        prev = np.ascontiguousarray(prev, dtype=np.float64)
        nxt = np.empty(g.n, np.float64)
        err, l1 = _f64(0), _f64(0)
        in_src = g.in_src if g.m else np.zeros(1, np.uint64)
        if self.lib.fo_ec_step(g.n, g.in_start, in_src, g.out_degree, damping, prev, nxt, C.byref(err), C.byref(l1)):
            raise ValueError("ec_step: invalid input")
        return nxt, err.value, l1.value

    def pagerank_fused_seq(self, g, damping=0.85, threshold=1e-15, max_iterations=10000,
                           norm=NORM_LINF, history_cap=0) -> Run:
        return self._run(self.lib.fo_pagerank_fused_seq, g, damping, threshold, max_iterations,
                         norm, (), history_cap)

    def pagerank_lockstep(self, g, wave_start, damping=0.85, threshold=1e-15,
                          max_iterations=10000, norm=NORM_LINF, history_cap=0) -> Run:
        ws = np.ascontiguousarray(wave_start, np.uint64)
        return self._run(self.lib.fo_pagerank_lockstep, g, damping, threshold, max_iterations,
                         norm, (len(ws) - 1, ws), history_cap)

    def dense_oracle(self, g, damping=0.85, threshold=1e-15, max_iterations=10000):
        ranks = np.empty(g.n, np.float64)
        in_src = g.in_src if g.m else np.zeros(1, np.uint64)
        rc = self.lib.fo_dense_oracle(g.n, g.in_start, in_src, g.out_degree, damping, threshold,
                                      max_iterations, ranks)
        if rc:
            raise ValueError("dense oracle: invalid input")
        return ranks

    def l1_norm(self, a, b) -> float:
        a = np.ascontiguousarray(a, np.float64)
        b = np.ascontiguousarray(b, np.float64)
        if a.shape != b.shape:
            raise ValueError(f"l1_norm: length mismatch ({len(a)} vs {len(b)})")
        return self.lib.fo_l1_norm(len(a), a, b)

    def linf_norm(self, a, b) -> float:
        a = np.ascontiguousarray(a, np.float64)
        b = np.ascontiguousarray(b, np.float64)
        if a.shape != b.shape:
            raise ValueError("linf_norm: length mismatch")
        return self.lib.fo_linf_norm(len(a), a, b)


ENGINES = {"ec_seq": 0, "fused_seq": 1, "ec_par": 2, "fused_par": 3}


class Reference:
    """ctypes binding of oracle/_ref/libfpr_ref.so (the reference itself)."""

    def __init__(self, path: str = REF_SO) -> None:
        L = C.CDLL(path)
        L.ref_last_error.restype = C.c_void_p
        L.ref_generate_rmat.argtypes = [C.c_uint32, _u64, _f64, _f64, _f64, _f64, _u64, _u64p, _u64p]
        L.ref_random_sparse.argtypes = [_u64, _u64, _u64, _u64p, _u64p]
        L.ref_random_sparse.restype = _u64
        L.ref_build_csr.argtypes = [_u64, _u64, _u64p, _u64p, _u64p, _u64p, _u64p, C.POINTER(_u64)]
        L.ref_graph_create.argtypes = [_u64, _u64, _u64p, _u64p, _u64p]
        L.ref_graph_create.restype = C.c_void_p
        L.ref_graph_destroy.argtypes = [C.c_void_p]
        L.ref_graph_run.argtypes = [C.c_void_p, C.c_int, _f64, _f64, _u64, C.c_uint, _f64p, _f64p,
                                    C.POINTER(_u64), C.POINTER(C.c_int), C.POINTER(_f64),
                                    C.POINTER(_f64)]
        L.ref_dense_oracle.argtypes = [_u64, _u64, _u64p, _u64p, _u64p, _f64, _f64, _u64, _f64p]
        L.ref_last_error_len.restype = _u64
        L.ref_parse_edge_list.argtypes = [C.c_char_p, _u64, C.POINTER(_u64), C.POINTER(_u64), C.c_void_p,
                                          _u64, C.POINTER(_u64)]
        self.lib = L

    def parse_edge_list(self, text: bytes) -> Parsed:
        """fpr::parse_edge_list itself (edge_list.hpp:39-80)."""
        n, m, line = _u64(0), _u64(0), _u64(0)
        rc = self.lib.ref_parse_edge_list(text, len(text), C.byref(n), C.byref(m), None, 0, C.byref(line))
        if rc == 3:
            what = C.string_at(self.lib.ref_last_error(), self.lib.ref_last_error_len())
            return Parsed(0, np.zeros((0, 2), np.uint64), line.value, what.decode("latin-1"))
        if rc:
            raise RuntimeError(self._err())
        edges = np.empty((max(m.value, 1), 2), np.uint64)
        rc = self.lib.ref_parse_edge_list(text, len(text), C.byref(n), C.byref(m), edges.ctypes.data,
                                          m.value, C.byref(line))
        assert rc == 0
        return Parsed(n.value, edges[: m.value].copy())

    def _err(self) -> str:
        return C.string_at(self.lib.ref_last_error()).decode()

    def generate_rmat(self, scale, edge_factor, a=0.57, b=0.19, c=0.19, d=0.05, seed=0):
        draws = edge_factor << scale
        src = np.empty(draws, np.uint64)
        dst = np.empty(draws, np.uint64)
        if self.lib.ref_generate_rmat(scale, edge_factor, a, b, c, d, seed, src, dst):
            raise ValueError(self._err())
        return 1 << scale, src, dst

    def random_sparse(self, n, avg_degree, seed):
        src = np.empty(n * avg_degree, np.uint64)
        dst = np.empty(n * avg_degree, np.uint64)
        k = self.lib.ref_random_sparse(n, avg_degree, seed, src, dst)
        return n, src[:k].copy(), dst[:k].copy()

    def build_csr(self, n, src, dst) -> Graph:
        src = np.ascontiguousarray(src, np.uint64)
        dst = np.ascontiguousarray(dst, np.uint64)
        in_start = np.empty(n + 1, np.uint64)
        in_src = np.empty(max(len(src), 1), np.uint64)
        out_degree = np.empty(max(n, 1), np.uint64)
        m = _u64(0)
        if self.lib.ref_build_csr(n, len(src), src, dst, in_start, in_src, out_degree, C.byref(m)):
            raise ValueError(self._err())
        return Graph(n, m.value, in_start, in_src[: m.value].copy(), out_degree[:n].copy())

    def run(self, g: Graph, engine: str, damping=0.85, threshold=1e-15, max_iterations=10000,
            threads=1, handle=None) -> Run:
        own = handle is None
        in_src = g.in_src if g.m else np.zeros(1, np.uint64)
        h = handle or self.lib.ref_graph_create(g.n, g.m, g.in_start, in_src, g.out_degree)
        try:
            ranks = np.empty(max(g.n, 1), np.float64)
            errors = np.empty(max_iterations, np.float64)
            it, conv, fe, secs = _u64(0), C.c_int(0), _f64(0), _f64(0)
            rc = self.lib.ref_graph_run(h, ENGINES[engine], damping, threshold, max_iterations,
                                        threads, ranks, errors, C.byref(it), C.byref(conv),
                                        C.byref(fe), C.byref(secs))
            if rc:
                raise ValueError(self._err())
            k = it.value
            return Run(ranks[: g.n], errors[:k].copy(), None, k, None, secs.value)
        finally:
            if own:
                self.lib.ref_graph_destroy(h)

    def graph_handle(self, g: Graph):
        in_src = g.in_src if g.m else np.zeros(1, np.uint64)
        return self.lib.ref_graph_create(g.n, g.m, g.in_start, in_src, g.out_degree)

    def destroy(self, h) -> None:
        self.lib.ref_graph_destroy(h)

    def dense_oracle(self, g, damping=0.85, threshold=1e-15, max_iterations=10000):
        ranks = np.empty(g.n, np.float64)
        in_src = g.in_src if g.m else np.zeros(1, np.uint64)
        if self.lib.ref_dense_oracle(g.n, g.m, g.in_start, in_src, g.out_degree, damping,
                                     threshold, max_iterations, ranks):
            raise ValueError(self._err())
        return ranks


def load_reference() -> Reference | None:
    return Reference() if os.path.exists(REF_SO) else None
