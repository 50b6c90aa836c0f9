"""B200-native FusEd-PageRank (arXiv 2203.09284) -- Python host mirror.

Mirrors the reference's engine interface (``/root/reference/proj/include/fpr``):
``PageRankConfig`` (pagerank.hpp:17-22), ``PageRankResult`` = ``RankVector`` +
``ConvergenceTrace`` (:24-38), ``Graph`` (graph.hpp:20-30), ``RmatParams``
(rmat.hpp:14-22), ``EngineKind`` tags (metrics.hpp:14-35) and ``l1_norm`` /
``linf_norm`` (metrics.hpp:54-75).  The engines are the GPU ones:

    pagerank_ec_b200(g, cfg)              ~ pagerank_ec_seq / pagerank_ec_par
    pagerank_fused_b200(g, cfg)           ~ pagerank_fused_par (block-async GS)
    pagerank_fused_lockstep_b200(g, cfg)  ~ deterministic wave-lockstep GS

Every call goes through the C ABI of ``libfpr_b200.so`` (include/fpr_b200.h).
There is no CPU fallback: if the library is missing or no B200 is present the
call raises.  Argument errors raise ``ValueError`` carrying the reference's
``std::invalid_argument`` text.
"""
from __future__ import annotations

import ctypes as C
import enum
import os
from dataclasses import dataclass, field

import numpy as np

__all__ = [
    "PageRankConfig", "RankVector", "ConvergenceTrace", "PageRankResult", "Graph", "RmatParams",
    "EngineKind", "DeviceGraph", "B200Error", "pagerank_ec_b200", "pagerank_fused_b200",
    "pagerank_fused_lockstep_b200", "run_engine", "l1_norm", "linf_norm", "to_string",
    "parse_engine", "lib", "LIB_PATH", "EdgeSet", "ParseError", "parse_edge_list", "write_edge_list",
    "build_csr",
]

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("FPR_B200_LIB") or os.path.join(HERE, "libfpr_b200.so")

OK, EINVAL, ECUDA, ENCCL, ENOMEM, ERANGE, EPARSE = 0, 1, 2, 3, 4, 5, 6
ENGINE_EC, ENGINE_FUSED, ENGINE_FUSED_LOCKSTEP = 0, 1, 2
NORM_LINF, NORM_L1 = 0, 1
GEN_RMAT, GEN_UNIFORM, GEN_CHUNGLU = 0, 1, 2
OPT_REORDER = 1  # FPR_B200_OPT_REORDER
OPT_PB = 4  # FPR_B200_OPT_PB: force propagation-blocked sweeps
OPT_PULL = 16  # FPR_B200_OPT_PULL: force pull sweeps (default: the library picks, include/fpr_b200.h)
SWEEP_PULL, SWEEP_PB = 0, 1  # fpr_b200_result.sweep
OPT_REORDER_SOURCES = 8  # FPR_B200_OPT_REORDER_SOURCES
OPT_REORDER_BLOCKS = 32  # FPR_B200_OPT_REORDER_BLOCKS


class B200Error(RuntimeError):
    def __init__(self, code: int, msg: str):
        super().__init__(msg)
        self.code = code


class ParseError(RuntimeError):
    """fpr::ParseError (edge_list.hpp:17-21): what() = "line L: ...",
    line_number = the 1-based line of the first malformed line."""

    def __init__(self, line_number: int, what: str):
        super().__init__(what)
        self.line_number = line_number


# ----------------------------------------------------------------- C structs
class _GraphView(C.Structure):
    _fields_ = [("n", C.c_uint64), ("m", C.c_uint64), ("in_start", C.c_void_p),
                ("in_src", C.c_void_p), ("out_degree", C.c_void_p)]


class _Config(C.Structure):
    _fields_ = [("damping", C.c_double), ("threshold", C.c_double),
                ("max_iterations", C.c_uint64), ("thread_count", C.c_uint32)]


class _Options(C.Structure):
    _fields_ = [("device", C.c_int32), ("norm", C.c_int32), ("wave_count", C.c_uint32),
                ("flags", C.c_uint32), ("stream", C.c_void_p), ("devices", C.POINTER(C.c_int32)),
                ("ndevices", C.c_uint32), ("reserved0", C.c_uint32)]


class _Result(C.Structure):
    _fields_ = [("iterations", C.c_uint64), ("converged", C.c_int32), ("sweep", C.c_int32),
                ("final_error", C.c_double), ("solve_ms", C.c_double), ("setup_ms", C.c_double),
                ("kernel_launches", C.c_uint64)]


class _GenParams(C.Structure):
    _fields_ = [("kind", C.c_int32), ("scale", C.c_uint32), ("edge_factor", C.c_uint64),
                ("a", C.c_double), ("b", C.c_double), ("c", C.c_double), ("d", C.c_double),
                ("n", C.c_uint64), ("avg_degree", C.c_uint64), ("seed", C.c_uint64),
                ("draws", C.c_uint64), ("alpha", C.c_double), ("kmax", C.c_uint64),
                ("relabel_bfs", C.c_int32), ("reserved0", C.c_int32), ("bfs_root", C.c_uint64)]


class _ParseErr(C.Structure):
    _fields_ = [("line", C.c_uint64), ("kind", C.c_int32), ("message_len", C.c_uint32),
                ("message", C.c_char * 256)]


EXPORTS = [
    "fpr_b200_options_init", "fpr_b200_config_init", "fpr_b200_last_error", "fpr_b200_version",
    "fpr_b200_graph_create", "fpr_b200_graph_generate", "fpr_b200_graph_destroy",
    "fpr_b200_graph_info", "fpr_b200_graph_download_csr", "fpr_b200_graph_wave_starts",
    "fpr_b200_run", "fpr_b200_graph_ranks_device", "fpr_b200_pagerank", "fpr_b200_graph_bfs_order",
    "fpr_b200_graph_validate", "fpr_b200_graph_partition", "fpr_b200_part_info",
    "fpr_b200_part_init", "fpr_b200_part_sweep", "fpr_b200_part_ranks",
    "fpr_b200_parse_edge_list", "fpr_b200_graph_from_edge_list", "fpr_b200_part_sweep_peers",
    "fpr_b200_ipc_export", "fpr_b200_ipc_import", "fpr_b200_ipc_close", "fpr_b200_graph_set_wave_count",
    "fpr_b200_graph_from_edges", "fpr_b200_part_ranks_prev", "fpr_b200_part_create",
    "fpr_b200_mgpu_create", "fpr_b200_mgpu_generate", "fpr_b200_mgpu_run", "fpr_b200_mgpu_info",
    "fpr_b200_mgpu_destroy", "fpr_b200_generate_edges", "fpr_b200_graph_layout_info",
    "fpr_b200_gate_bytes", "fpr_b200_gate_init", "fpr_b200_gate_update", "fpr_b200_gate_read",
    "fpr_b200_part_set_gate", "fpr_b200_part_ranks_after",
]

_lib = None


def lib() -> C.CDLL:
    """Load libfpr_b200.so (raises if it was not built -- no fallback)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise B200Error(ECUDA, f"{LIB_PATH} is not built; run __graft_entry__.build() "
                                   "(make -C paper_2203_09284_b200/csrc)")
        L = C.CDLL(LIB_PATH)
        vp, u64, i32 = C.c_void_p, C.c_uint64, C.c_int
        L.fpr_b200_last_error.restype = C.c_char_p
        L.fpr_b200_options_init.argtypes = [C.POINTER(_Options)]
        L.fpr_b200_config_init.argtypes = [C.POINTER(_Config)]
        L.fpr_b200_graph_create.argtypes = [C.POINTER(_GraphView), C.POINTER(_Options), C.POINTER(vp)]
        L.fpr_b200_graph_generate.argtypes = [C.POINTER(_GenParams), C.POINTER(_Options), C.POINTER(vp)]
        L.fpr_b200_graph_destroy.argtypes = [vp]
        L.fpr_b200_graph_destroy.restype = None
        L.fpr_b200_graph_info.argtypes = [vp, C.POINTER(u64), C.POINTER(u64), C.POINTER(u64)]
        L.fpr_b200_graph_layout_info.argtypes = [vp, C.POINTER(C.c_int), C.POINTER(u64), C.POINTER(u64),
                                                 C.POINTER(u64)]
        L.fpr_b200_graph_download_csr.argtypes = [vp, vp, vp, vp]
        L.fpr_b200_graph_wave_starts.argtypes = [vp, C.c_uint32, vp, u64, C.POINTER(u64)]
        L.fpr_b200_graph_bfs_order.argtypes = [vp, u64, vp]
        L.fpr_b200_graph_validate.argtypes = [vp, C.POINTER(C.c_uint32)]
        L.fpr_b200_run.argtypes = [vp, i32, C.POINTER(_Config), vp, vp, vp, vp, u64, C.POINTER(_Result)]
        L.fpr_b200_graph_ranks_device.argtypes = [vp]
        L.fpr_b200_graph_ranks_device.restype = vp
        L.fpr_b200_pagerank.argtypes = [C.POINTER(_GraphView), i32, C.POINTER(_Config),
                                        C.POINTER(_Options), vp, vp, u64, C.POINTER(_Result)]
        # Every pointer-taking entry point gets its argtypes here, once: an
        # unset argtype makes ctypes pass a Python int as a 32-bit C int.
        u32 = C.c_uint32
        L.fpr_b200_graph_partition.argtypes = [vp, u32, u32, C.POINTER(_Options), vp, C.POINTER(u64),
                                               C.POINTER(vp)]
        L.fpr_b200_part_create.argtypes = [C.POINTER(_GraphView), u32, u32, C.POINTER(_Options), vp,
                                           C.POINTER(u64), C.POINTER(vp)]
        L.fpr_b200_part_info.argtypes = [vp, C.POINTER(u64), C.POINTER(u64), C.POINTER(u64), C.POINTER(u32),
                                         C.POINTER(u32)]
        L.fpr_b200_part_init.argtypes = [vp, vp]
        L.fpr_b200_part_sweep.argtypes = [vp, i32, C.POINTER(_Config), vp, vp, vp]
        L.fpr_b200_part_sweep_peers.argtypes = [vp, i32, C.POINTER(_Config), vp, vp, vp, u32, vp]
        L.fpr_b200_part_ranks.argtypes = [vp, vp]
        L.fpr_b200_part_ranks_prev.argtypes = [vp, vp]
        L.fpr_b200_gate_bytes.argtypes = [u64]
        L.fpr_b200_gate_bytes.restype = u64
        L.fpr_b200_gate_init.argtypes = [vp, u64, i32, vp]
        L.fpr_b200_gate_update.argtypes = [vp, vp, u32, C.POINTER(_Config), i32, i32, vp]
        L.fpr_b200_gate_read.argtypes = [vp, i32, vp, C.POINTER(u64), C.POINTER(C.c_int), vp, vp, u64]
        L.fpr_b200_part_set_gate.argtypes = [vp, vp]
        L.fpr_b200_part_ranks_after.argtypes = [vp, u64, vp]
        L.fpr_b200_ipc_export.argtypes = [vp, vp]
        L.fpr_b200_ipc_import.argtypes = [C.c_char_p, i32, C.POINTER(vp)]
        L.fpr_b200_ipc_close.argtypes = [vp]
        L.fpr_b200_graph_set_wave_count.argtypes = [vp, u32]
        L.fpr_b200_graph_from_edges.argtypes = [u64, u64, vp, vp, C.POINTER(_Options), C.POINTER(vp)]
        L.fpr_b200_parse_edge_list.argtypes = [vp, u64, C.POINTER(_Options), C.POINTER(u64),
                                               C.POINTER(u64), vp, u64, C.POINTER(_ParseErr)]
        L.fpr_b200_graph_from_edge_list.argtypes = [vp, u64, C.POINTER(_Options), C.POINTER(vp),
                                                    C.POINTER(_ParseErr)]
        L.fpr_b200_mgpu_create.argtypes = [C.POINTER(_GraphView), C.POINTER(_Options), C.POINTER(vp)]
        L.fpr_b200_mgpu_generate.argtypes = [C.POINTER(_GenParams), C.POINTER(_Options), C.POINTER(vp)]
        L.fpr_b200_mgpu_run.argtypes = [vp, i32, C.POINTER(_Config), vp, vp, vp, u64, C.POINTER(_Result)]
        L.fpr_b200_mgpu_info.argtypes = [vp, C.POINTER(u64), C.POINTER(u64), C.POINTER(u32), vp]
        L.fpr_b200_generate_edges.argtypes = [C.POINTER(_GenParams), C.POINTER(_Options), vp, vp, u64,
                                              C.POINTER(u64)]
        L.fpr_b200_mgpu_destroy.argtypes = [vp]
        L.fpr_b200_mgpu_destroy.restype = None
        _lib = L
    return _lib


def _check(rc: int, perr: "_ParseErr | None" = None) -> None:
    if rc == EPARSE and perr is not None:
        raise ParseError(int(perr.line), perr.message.decode("latin-1"))
    if rc != OK:
        msg = lib().fpr_b200_last_error().decode()
        if rc in (EINVAL, ERANGE):
            raise ValueError(msg)
        raise B200Error(rc, msg)


# ------------------------------------------------------- reference mirrors
@dataclass
class PageRankConfig:
    """fpr::PageRankConfig (pagerank.hpp:17-22)."""

    damping: float = 0.85
    threshold: float = 1e-15
    max_iterations: int = 10000
    thread_count: int = 1  # validated; the GPU engines ignore it

    def _c(self) -> _Config:
        return _Config(self.damping, self.threshold, self.max_iterations, self.thread_count)


@dataclass
class RankVector:
    values: np.ndarray
    final_error: float = 1.0


@dataclass
class ConvergenceTrace:
    errors: np.ndarray
    iterations: int = 0
    converged: bool = False
    l1_errors: np.ndarray | None = None  # extension: sum |delta| per iteration
    iter_ns: np.ndarray | None = None    # extension: device ns per iteration


@dataclass
class PageRankResult:
    ranks: RankVector
    trace: ConvergenceTrace
    solve_ms: float = 0.0
    kernel_launches: int = 0
    setup_ms: float = 0.0  # device time before the first sweep (init; one-time layouts on first use)
    sweep: int = SWEEP_PULL  # sweep kind that ran (SWEEP_PULL / SWEEP_PB)


@dataclass
class Graph:
    """fpr::Graph (graph.hpp:20-30): in-CSR with u64 arrays."""

    n: int
    m: int
    in_start: np.ndarray
    in_src: np.ndarray
    out_degree: np.ndarray

    def in_degree(self, u=None):
        d = np.diff(self.in_start)
        return d if u is None else int(d[u])


@dataclass
class RmatParams:
    """fpr::RmatParams (rmat.hpp:14-22)."""

    scale: int = 10
    edge_factor: int = 20
    a: float = 0.57
    b: float = 0.19
    c: float = 0.19
    d: float = 0.05
    seed: int = 0


class EngineKind(enum.Enum):
    """metrics.hpp:14 EngineKind + the B200 engines."""

    EcSeq = "ec_seq"
    FusedSeq = "fused_seq"
    EcPar = "ec_par"
    FusedPar = "fused_par"
    EcB200 = "ec_b200"
    FusedB200 = "fused_b200"
    FusedLockstepB200 = "fused_lockstep_b200"


def to_string(kind: EngineKind) -> str:
    return kind.value


def parse_engine(name: str) -> EngineKind:
    for k in EngineKind:
        if k.value == name:
            return k
    raise ValueError(f"unknown engine tag '{name}' (expected "
                     + "|".join(k.value for k in EngineKind) + ")")


_B200_ENGINE = {EngineKind.EcB200: ENGINE_EC, EngineKind.FusedB200: ENGINE_FUSED,
                EngineKind.FusedLockstepB200: ENGINE_FUSED_LOCKSTEP}


CUDA_STREAM_LEGACY = 1  # cudaStreamLegacy


def torch_stream_handle() -> int:
    """cudaStream_t of torch's current stream for fpr_b200_options.stream.
    torch reports its default stream as 0, which the C ABI reads as "make a
    library stream"; map it to cudaStreamLegacy so the library's work is
    ordered with torch's kernels, events and NCCL collectives."""
    import torch

    h = torch.cuda.current_stream().cuda_stream
    return h if h else CUDA_STREAM_LEGACY


def _options(device=-1, norm=NORM_LINF, wave_count=0, stream=None, reorder=False, pb=None) -> _Options:
    o = _Options()
    lib().fpr_b200_options_init(C.byref(o))
    o.device = device
    o.norm = norm
    o.wave_count = wave_count
    # reorder: False, True / "degree" (FPR_B200_OPT_REORDER) or "sources"
    # (FPR_B200_OPT_REORDER_SOURCES)
    if reorder not in (False, True, "degree", "sources", "blocks"):
        raise ValueError(f"reorder must be False, True, 'degree', 'sources' or 'blocks', not {reorder!r}")
    ro = {"sources": OPT_REORDER_SOURCES, "blocks": OPT_REORDER_BLOCKS}.get(reorder, OPT_REORDER if reorder else 0)
    # pb: None = the library picks the sweep kind, True = propagation-blocked, False = pull
    o.flags = ro | (0 if pb is None else (OPT_PB if pb else OPT_PULL))
    o.stream = stream
    return o


def _u64(a) -> np.ndarray:
    return np.ascontiguousarray(a, dtype=np.uint64)


class DeviceGraph:
    """A graph resident in HBM (int64 offsets, int32 ids) + its task partition."""

    def __init__(self, handle: int, device=-1, norm=NORM_LINF, wave_count=0):
        self._h = C.c_void_p(handle)
        self.norm = norm
        n, m, nt = C.c_uint64(), C.c_uint64(), C.c_uint64()
        _check(lib().fpr_b200_graph_info(self._h, C.byref(n), C.byref(m), C.byref(nt)))
        self.n, self.m, self.ntasks = n.value, m.value, nt.value

    # -- construction ---------------------------------------------------
    @classmethod
    def from_graph(cls, g: Graph, device=-1, norm=NORM_LINF, wave_count=0, stream=None, reorder=False,
                   pb=None):
        ins, src, od = _u64(g.in_start), _u64(g.in_src), _u64(g.out_degree)
        v = _GraphView(g.n, g.m, ins.ctypes.data, src.ctypes.data if g.m else None, od.ctypes.data)
        h = C.c_void_p()
        _check(lib().fpr_b200_graph_create(C.byref(v), C.byref(_options(device, norm, wave_count, stream, reorder, pb)),
                                           C.byref(h)))
        return cls(h.value, device, norm, wave_count)

    @classmethod
    def _generate(cls, gp, device, norm, wave_count, stream, reorder=False, pb=None):
        h = C.c_void_p()
        _check(lib().fpr_b200_graph_generate(C.byref(gp), C.byref(_options(device, norm, wave_count, stream, reorder, pb)),
                                             C.byref(h)))
        return cls(h.value, device, norm, wave_count)

    @classmethod
    def generate_rmat(cls, p: RmatParams, device=-1, norm=NORM_LINF, wave_count=0, stream=None,
                      relabel_bfs=False, bfs_root=0, reorder=False, pb=None):
        """build_csr(generate_rmat(p)) on the device; relabel_bfs=True gives
        BASELINE config 3's crawl order (BFS from bfs_root over out-edges)."""
        gp = _GenParams(GEN_RMAT, p.scale, p.edge_factor, p.a, p.b, p.c, p.d, 0, 0, p.seed,
                        0, 0.0, 0, int(relabel_bfs), 0, bfs_root)
        return cls._generate(gp, device, norm, wave_count, stream, reorder, pb)

    @classmethod
    def generate_uniform(cls, n: int, avg_degree: int, seed: int, device=-1, norm=NORM_LINF,
                         wave_count=0, stream=None, reorder=False, pb=None):
        """build_csr(testutil::random_sparse(n, avg_degree, SplitMix64(seed)))."""
        gp = _GenParams(GEN_UNIFORM, 0, 0, 0.0, 0.0, 0.0, 0.0, n, avg_degree, seed)
        return cls._generate(gp, device, norm, wave_count, stream, reorder, pb)

    @classmethod
    def generate_chunglu(cls, n: int, draws: int, seed: int, alpha: float = 2.1, kmax: int = 1_000_000,
                         device=-1, norm=NORM_LINF, wave_count=0, stream=None, reorder=False, pb=None):
        """BASELINE config 4 (definition: DESIGN.md §4.1; oracle fo_generate_chunglu)."""
        gp = _GenParams(GEN_CHUNGLU, 0, 0, 0.0, 0.0, 0.0, 0.0, n, 0, seed, draws, alpha, kmax)
        return cls._generate(gp, device, norm, wave_count, stream, reorder, pb)

    @classmethod
    def from_edges(cls, n: int, src, dst, device=-1, norm=NORM_LINF, wave_count=0, stream=None, reorder=False,
                   pb=None):
        """fpr::build_csr(EdgeSet{n, (src, dst)}) on the device (graph.hpp:35-70):
        duplicates and self-loops dropped, in-segments ascending; ValueError
        names the first out-of-range edge as build_csr does."""
        s_, d_ = _u64(src), _u64(dst)
        if len(s_) != len(d_):
            raise ValueError("from_edges: src and dst lengths differ")
        h = C.c_void_p()
        L = lib()
        _check(L.fpr_b200_graph_from_edges(n, len(s_), s_.ctypes.data if len(s_) else None,
                                           d_.ctypes.data if len(d_) else None,
                                           C.byref(_options(device, norm, wave_count, stream, reorder, pb)),
                                           C.byref(h)))
        return cls(h.value, device, norm, wave_count)

    @classmethod
    def from_edge_list(cls, text, device=-1, norm=NORM_LINF, wave_count=0, stream=None, reorder=False,
                       pb=None):
        """build_csr(parse_edge_list(text)) -- parsing, id compaction and the
        CSR build all on the device (edge_list.hpp:39-80, graph.hpp:35-70)."""
        ptr, nbytes, keep = _text_arg(text)
        h = C.c_void_p()
        perr = _ParseErr()
        _check(lib().fpr_b200_graph_from_edge_list(ptr, nbytes, C.byref(_options(device, norm, wave_count,
                                                                                stream, reorder, pb)),
                                                   C.byref(h), C.byref(perr)), perr)
        del keep
        return cls(h.value, device, norm, wave_count)

    def set_wave_count(self, waves: int) -> None:
        """Lockstep engine: waves per sweep for later runs (0 = auto)."""
        _check(lib().fpr_b200_graph_set_wave_count(self._h, waves))

    def validate(self) -> int:
        """0 iff the resident CSR satisfies build_csr's invariants (device check)."""
        f = C.c_uint32()
        _check(lib().fpr_b200_graph_validate(self._h, C.byref(f)))
        return f.value

    def bfs_order(self, root: int = 0) -> np.ndarray:
        out = np.empty(self.n, np.uint64)
        _check(lib().fpr_b200_graph_bfs_order(self._h, root, out.ctypes.data))
        return out

    def close(self) -> None:
        if self._h:
            lib().fpr_b200_graph_destroy(self._h)
            self._h = C.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def __enter__(self):
        return self

    def __exit__(self, *a):
        self.close()

    # -- queries ----------------------------------------------------------
    def download(self) -> Graph:
        ins = np.empty(self.n + 1, np.uint64)
        src = np.empty(max(self.m, 1), np.uint64)
        od = np.empty(max(self.n, 1), np.uint64)
        _check(lib().fpr_b200_graph_download_csr(self._h, ins.ctypes.data, src.ctypes.data, od.ctypes.data))
        return Graph(self.n, self.m, ins, src[: self.m], od[: self.n])

    def download_into(self, in_start: np.ndarray, in_src: np.ndarray, out_degree: np.ndarray) -> None:
        """download() into caller-owned u64 arrays (e.g. pinned views)."""
        for a, k in ((in_start, self.n + 1), (in_src, self.m), (out_degree, self.n)):
            if a.dtype != np.uint64 or not a.flags.c_contiguous or len(a) < k:
                raise ValueError("download_into: need C-contiguous u64 arrays of n+1, m and n entries")
        _check(lib().fpr_b200_graph_download_csr(self._h, in_start.ctypes.data, in_src.ctypes.data if self.m else None,
                                                 out_degree.ctypes.data))

    def layout_info(self) -> dict:
        """Propagation-blocked layout sizes (0 until the first PB solve built it)."""
        sw, runs, pieces, tiles = C.c_int(), C.c_uint64(), C.c_uint64(), C.c_uint64()
        _check(lib().fpr_b200_graph_layout_info(self._h, C.byref(sw), C.byref(runs), C.byref(pieces),
                                                C.byref(tiles)))
        return {"sweep": sw.value, "runs": runs.value, "pieces": pieces.value, "tiles": tiles.value}

    def wave_starts(self, wave_count: int = 0) -> np.ndarray:
        nw = C.c_uint64()
        _check(lib().fpr_b200_graph_wave_starts(self._h, wave_count, None, 0, C.byref(nw)))
        out = np.empty(nw.value + 1, np.uint64)
        _check(lib().fpr_b200_graph_wave_starts(self._h, wave_count, out.ctypes.data, len(out), C.byref(nw)))
        return out

    def ranks_device_ptr(self) -> int:
        return lib().fpr_b200_graph_ranks_device(self._h) or 0

    # -- engines ----------------------------------------------------------
    def run(self, engine: int, cfg: PageRankConfig, copy_ranks=True, copy_trace=True) -> PageRankResult:
        cap = int(cfg.max_iterations) if copy_trace else 0
        cap = min(cap, 1 << 24)
        errors = np.empty(max(cap, 1), np.float64)
        l1 = np.empty(max(cap, 1), np.float64)
        ns = np.empty(max(cap, 1), np.uint64)
        ranks = np.empty(max(self.n, 1), np.float64) if copy_ranks else None
        res = _Result()
        c = cfg._c()
        _check(lib().fpr_b200_run(self._h, engine, C.byref(c),
                                  ranks.ctypes.data if copy_ranks else None,
                                  errors.ctypes.data if copy_trace else None,
                                  l1.ctypes.data if copy_trace else None,
                                  ns.ctypes.data if copy_trace else None, cap, C.byref(res)))
        k = res.iterations
        trace = ConvergenceTrace(errors[:k].copy() if copy_trace else np.empty(0), k, bool(res.converged),
                                 l1[:k].copy() if copy_trace else None, ns[:k].copy() if copy_trace else None)
        rv = RankVector(ranks[: self.n] if copy_ranks else np.empty(0), res.final_error)
        return PageRankResult(rv, trace, res.solve_ms, res.kernel_launches, res.setup_ms, res.sweep)


class MultiDeviceGraph:
    """A graph split by destination range over several devices, driven from
    this thread (fpr_b200_mgpu_*): part r on devices[r]; devices may repeat
    (parts sharing a GPU run one after the other)."""

    def __init__(self, handle: int, devices):
        self._h = C.c_void_p(handle)
        self.devices = list(devices)
        n, m, p = C.c_uint64(), C.c_uint64(), C.c_uint32()
        _check(lib().fpr_b200_mgpu_info(self._h, C.byref(n), C.byref(m), C.byref(p), None))
        self.n, self.m, self.nparts = n.value, m.value, p.value
        b = np.empty(self.nparts + 1, np.uint64)
        _check(lib().fpr_b200_mgpu_info(self._h, None, None, None, b.ctypes.data))
        self.bounds = b

    @staticmethod
    def _opts(devices, norm, keep, pb=None):
        arr = (C.c_int32 * len(devices))(*devices)
        keep.append(arr)
        o = _options(norm=norm, pb=pb)
        o.devices = C.cast(arr, C.POINTER(C.c_int32))
        o.ndevices = len(devices)
        return o

    @classmethod
    def from_graph(cls, g: Graph, devices, norm=NORM_LINF, pb=None):
        keep = []
        ins, src, od = _u64(g.in_start), _u64(g.in_src), _u64(g.out_degree)
        v = _GraphView(g.n, g.m, ins.ctypes.data, src.ctypes.data if g.m else None, od.ctypes.data)
        h = C.c_void_p()
        _check(lib().fpr_b200_mgpu_create(C.byref(v), C.byref(cls._opts(devices, norm, keep, pb)), C.byref(h)))
        return cls(h.value, devices)

    @classmethod
    def generate_rmat(cls, p: RmatParams, devices, norm=NORM_LINF, pb=None):
        keep = []
        gp = _GenParams(GEN_RMAT, p.scale, p.edge_factor, p.a, p.b, p.c, p.d, 0, 0, p.seed, 0, 0.0, 0, 0, 0, 0)
        h = C.c_void_p()
        _check(lib().fpr_b200_mgpu_generate(C.byref(gp), C.byref(cls._opts(devices, norm, keep, pb)), C.byref(h)))
        return cls(h.value, devices)

    def run(self, engine: int, cfg: PageRankConfig, copy_ranks=True, copy_trace=True) -> PageRankResult:
        cap = min(int(cfg.max_iterations), 1 << 24) if copy_trace else 0
        errors = np.empty(max(cap, 1), np.float64)
        l1 = np.empty(max(cap, 1), np.float64)
        ranks = np.empty(max(self.n, 1), np.float64) if copy_ranks else None
        res = _Result()
        c = cfg._c()
        _check(lib().fpr_b200_mgpu_run(self._h, engine, C.byref(c), ranks.ctypes.data if copy_ranks else None,
                                       errors.ctypes.data if copy_trace else None,
                                       l1.ctypes.data if copy_trace else None, cap, C.byref(res)))
        k = res.iterations
        trace = ConvergenceTrace(errors[:k].copy() if copy_trace else np.empty(0), k, bool(res.converged),
                                 l1[:k].copy() if copy_trace else None, None)
        rv = RankVector(ranks[: self.n] if copy_ranks else np.empty(0), res.final_error)
        return PageRankResult(rv, trace, res.solve_ms, res.kernel_launches, res.setup_ms, res.sweep)

    def close(self) -> None:
        if self._h:
            lib().fpr_b200_mgpu_destroy(self._h)
            self._h = C.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def __enter__(self):
        return self

    def __exit__(self, *a):
        self.close()


def generate_edges(kind: str, device=-1, **p) -> "EdgeSet":
    """The generator's EdgeSet before build_csr, in generation order, drawn on
    the device: kind "rmat" (RmatParams fields: fpr::generate_rmat, rmat.hpp:
    42-77, self-loops and duplicates kept) or "uniform" (n, avg_degree, seed:
    testutil::random_sparse, self-loops skipped)."""
    if kind == "rmat":
        r = p["params"]
        gp = _GenParams(GEN_RMAT, r.scale, r.edge_factor, r.a, r.b, r.c, r.d, 0, 0, r.seed)
        n = 1 << r.scale
    elif kind == "uniform":
        gp = _GenParams(GEN_UNIFORM, 0, 0, 0.0, 0.0, 0.0, 0.0, p["n"], p["avg_degree"], p["seed"])
        n = p["n"]
    else:
        raise ValueError("generate_edges: kind is 'rmat' or 'uniform'")
    o = _options(device=device)
    cnt = C.c_uint64()
    _check(lib().fpr_b200_generate_edges(C.byref(gp), C.byref(o), None, None, 0, C.byref(cnt)))
    e = np.empty((max(cnt.value, 1), 2), np.uint64)
    src = np.empty(max(cnt.value, 1), np.uint64)
    dst = np.empty(max(cnt.value, 1), np.uint64)
    _check(lib().fpr_b200_generate_edges(C.byref(gp), C.byref(o), src.ctypes.data, dst.ctypes.data, cnt.value,
                                         C.byref(cnt)))
    e[:, 0], e[:, 1] = src, dst
    return EdgeSet(n, e[: cnt.value])


def run_engine(kind: EngineKind | str, g, cfg: PageRankConfig, **kw) -> PageRankResult:
    """Run a B200 engine on a host ``Graph`` (uploaded, like the reference's
    by-reference Graph) or a resident ``DeviceGraph``."""
    if isinstance(kind, str):
        kind = parse_engine(kind)
    if kind not in _B200_ENGINE:
        raise ValueError(f"{kind.value} is a reference CPU engine, not a B200 engine")
    if isinstance(g, DeviceGraph):
        return g.run(_B200_ENGINE[kind], cfg)
    if g.n == 0:  # init_ranks (pagerank.hpp:56), checked before any device work
        c = cfg._c()
        _validate(c)
        raise ValueError("pagerank: graph has no vertices")
    with DeviceGraph.from_graph(g, **kw) as dg:
        return dg.run(_B200_ENGINE[kind], cfg)


def _validate(c: _Config) -> None:
    if not (c.damping > 0.0 and c.damping < 1.0):
        raise ValueError("pagerank: damping must be in (0,1)")
    if not (c.threshold > 0.0):
        raise ValueError("pagerank: threshold must be positive")
    if c.max_iterations == 0:
        raise ValueError("pagerank: max_iterations must be positive")
    if c.thread_count == 0:
        raise ValueError("pagerank: thread_count must be positive")


def pagerank_ec_b200(g, cfg: PageRankConfig | None = None, **kw) -> PageRankResult:
    return run_engine(EngineKind.EcB200, g, cfg or PageRankConfig(), **kw)


def pagerank_fused_b200(g, cfg: PageRankConfig | None = None, **kw) -> PageRankResult:
    return run_engine(EngineKind.FusedB200, g, cfg or PageRankConfig(), **kw)


def pagerank_fused_lockstep_b200(g, cfg: PageRankConfig | None = None, **kw) -> PageRankResult:
    return run_engine(EngineKind.FusedLockstepB200, g, cfg or PageRankConfig(), **kw)


def l1_norm(a, b) -> float:
    """metrics.hpp:54-62 (host-side metric, not the hot path)."""
    a = np.asarray(a, np.float64)
    b = np.asarray(b, np.float64)
    if a.shape != b.shape:
        raise ValueError(f"l1_norm: length mismatch ({a.size} vs {b.size})")
    return float(np.abs(a - b).sum())


def linf_norm(a, b) -> float:
    """metrics.hpp:68-75."""
    a = np.asarray(a, np.float64)
    b = np.asarray(b, np.float64)
    if a.shape != b.shape:
        raise ValueError("linf_norm: length mismatch")
    return float(np.abs(a - b).max()) if a.size else 0.0


# ------------------------------------------------------------ edge-list ingest
@dataclass
class EdgeSet:
    """fpr::EdgeSet (edge_set.hpp): n vertices, edges (m, 2) u64 (src, dst)."""

    n: int
    edges: np.ndarray


def _text_arg(text):
    """(pointer-compatible object, byte length).  bytes/str are passed as is;
    a contiguous numpy uint8 array (e.g. a view of pinned memory) by address,
    so a pinned buffer takes the direct-DMA path."""
    if isinstance(text, str):
        text = text.encode("latin-1")
    if isinstance(text, np.ndarray):
        a = np.ascontiguousarray(text).view(np.uint8).reshape(-1)
        return (a.ctypes.data if a.size else None), a.size, a
    if not isinstance(text, bytes):
        text = bytes(text)
    return text, len(text), text


def parse_edge_list(text, device: int = -1) -> EdgeSet:
    """fpr::parse_edge_list (edge_list.hpp:39-80) on the GPU: '#'/'%' comment
    and blank lines skipped, "src dst" decimal u64 pairs, sparse ids compacted
    to [0, n) in first-appearance order.  Raises ParseError for the first
    malformed line, with the reference's line number and message."""
    ptr, nbytes, keep = _text_arg(text)
    n, m = C.c_uint64(), C.c_uint64()
    perr = _ParseErr()
    opts = _options(device)
    L = lib()
    # Upper bound on edges: one per line.  One device pass when it suffices.
    cap = (nbytes + 3) // 4 + 1 if nbytes < (1 << 28) else 0
    edges = np.empty((max(cap, 1), 2), np.uint64)
    rc = L.fpr_b200_parse_edge_list(ptr, nbytes, C.byref(opts), C.byref(n), C.byref(m),
                                    edges.ctypes.data if cap else None, cap, C.byref(perr))
    if rc == ERANGE and m.value > cap or (rc == OK and not cap and m.value):
        edges = np.empty((m.value, 2), np.uint64)
        rc = L.fpr_b200_parse_edge_list(ptr, nbytes, C.byref(opts), C.byref(n), C.byref(m),
                                        edges.ctypes.data, m.value, C.byref(perr))
    _check(rc, perr)
    del keep
    return EdgeSet(n.value, edges[: m.value].copy() if cap else edges[: m.value])


def write_edge_list(es: EdgeSet, header=()) -> bytes:
    """fpr::write_edge_list (edge_list.hpp:84-89): '# ' + each header line,
    then one "src dst" line per edge.  Host-side formatting (vectorised), the
    inverse of parse_edge_list for densely labelled inputs."""
    head = "".join(f"# {h}\n" for h in header).encode()
    e = np.asarray(es.edges, dtype=np.uint64).reshape(-1, 2)
    if len(e) == 0:
        return head
    body = np.char.add(np.char.add(e[:, 0].astype(str), " "), e[:, 1].astype(str))
    return head + ("\n".join(body.tolist()) + "\n").encode()


def build_csr(n: int, src, dst, device: int = -1) -> Graph:
    """fpr::build_csr on the GPU, returned as host u64 arrays (fpr::Graph)."""
    with DeviceGraph.from_edges(n, src, dst, device=device) as dg:
        return dg.download()

