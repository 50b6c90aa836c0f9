"""Multi-GPU destination-range partitioning.

Each rank owns an edge-balanced range of destination rows (a merge-path split
of the n row ends + m edges) together with those rows' in-edges.  Source ids
are remapped into a padded exchange space of ``nparts * slice`` doubles
(``part(s) * slice + s - bounds[part(s)]``), so an iteration's only
communication is

  1. one equal-size all-gather of every part's contribution slice (NCCL over
     NVLink / NVSwitch when the backend is ``nccl``), and
  2. one all-gather of the per-part (max |delta|, sum |delta|) pairs, reduced
     in rank order on every rank (a deterministic L1 sum; the max is exact).

The stop rule is the reference's (``error <= threshold``, pagerank.hpp:141),
applied identically on every rank.  EC ping-pongs two exchange vectors
(Jacobi, bit-identical to one GPU up to the per-row reduction order); FUSED
updates one vector in place, so sources on the same GPU may be fresh and
remote ones are one exchange old -- block-asynchronous Gauss-Seidel at GPU
granularity, the ``pagerank_fused_par`` contract (pagerank.hpp:257-333).

The local sweep is pluggable: ``B200Part`` runs the sm_100a kernel through the
C ABI (``fpr_b200_part_*``); the gloo CPU tests plug in a numpy restatement.
The exchange is pluggable too: ``TorchExchange`` (torch.distributed, one
process per GPU) or ``EmulatedExchange`` (all parts in one process, slices
copied -- for single-GPU validation of the partitioned path).
"""
from __future__ import annotations

import ctypes as C
import time
from dataclasses import dataclass, field

import numpy as np

from . import (B200Error, DeviceGraph, PageRankConfig, _check, _Config, _options, lib, ENGINE_EC,
               ENGINE_FUSED, NORM_L1, NORM_LINF)


# ------------------------------------------------------------------ host logic
def partition_bounds(in_start: np.ndarray, nparts: int) -> np.ndarray:
    """Row bounds of the edge-balanced merge-path split (mirror of the device
    kernel part_bounds_kernel): part r owns rows [b[r], b[r+1])."""
    in_start = np.asarray(in_start, dtype=np.int64)
    n = len(in_start) - 1
    m = int(in_start[-1])
    total = n + m
    ends = in_start[1:] + np.arange(n, dtype=np.int64)  # merge position after row i's end marker
    b = np.empty(nparts + 1, dtype=np.int64)
    for r in range(nparts + 1):
        if r == nparts:
            b[r] = n
            continue
        diag = total * r // nparts
        # rows fully consumed at diag: count of i with in_start[i+1] <= diag - i - 1
        b[r] = int(np.searchsorted(ends + 1, diag, side="right"))
        b[r] = min(b[r], n)
    return b


def remap_sources(in_src: np.ndarray, bounds: np.ndarray, slice_: int) -> np.ndarray:
    """Global id -> padded exchange id (part(s) * slice + s - bounds[part(s)])."""
    s = np.asarray(in_src, dtype=np.int64)
    part = np.searchsorted(bounds[1:-1], s, side="right")
    return part * slice_ + (s - bounds[part])


# ------------------------------------------------------------------ exchanges
class TorchExchange:
    """One process per GPU: collectives through torch.distributed."""

    def __init__(self, group=None):
        import torch.distributed as dist

        self.dist = dist
        self.group = group
        self.rank = dist.get_rank(group)
        self.world = dist.get_world_size(group)

    def allgather_slices(self, buf, slice_: int):
        import torch

        mine = buf[self.rank * slice_:(self.rank + 1) * slice_]
        if buf.device.type == "cpu":  # gloo: no in-place aliasing
            mine = mine.clone()
        self.dist.all_gather_into_tensor(buf, mine, group=self.group)

    def allgather_pairs(self, pair):
        import torch

        out = torch.empty(2 * self.world, dtype=pair.dtype, device=pair.device)
        self.dist.all_gather_into_tensor(out, pair, group=self.group)
        return out


class EmulatedExchange:
    """All parts in one process (one GPU): slices copied between the parts'
    exchange vectors.  Validates partition + sweep + exchange on one device."""

    def __init__(self, nparts: int):
        self.world = nparts

    def allgather_slices_all(self, bufs, slice_: int):
        for r in range(self.world):
            src = bufs[r][r * slice_:(r + 1) * slice_]
            for q in range(self.world):
                if q != r:
                    bufs[q][r * slice_:(r + 1) * slice_].copy_(src)


# ------------------------------------------------------------------ local sweep
class B200Part:
    """This rank's part on its GPU, driven through the C ABI."""

    def __init__(self, full: DeviceGraph, nparts: int, part: int, device: int = 0, stream=None):
        self.nparts, self.part = nparts, part
        bounds = np.empty(nparts + 1, np.uint64)
        sl = C.c_uint64()
        h = C.c_void_p()
        L = lib()
        L.fpr_b200_graph_partition.argtypes = [C.c_void_p, C.c_uint32, C.c_uint32, C.c_void_p,
                                               C.c_void_p, C.POINTER(C.c_uint64), C.POINTER(C.c_void_p)]
        L.fpr_b200_part_init.argtypes = [C.c_void_p, C.c_void_p]
        L.fpr_b200_part_sweep.argtypes = [C.c_void_p, C.c_int, C.POINTER(_Config), C.c_void_p,
                                          C.c_void_p, C.c_void_p]
        L.fpr_b200_part_ranks.argtypes = [C.c_void_p, C.c_void_p]
        opts = _options(device=device, stream=stream)
        _check(L.fpr_b200_graph_partition(full._h, nparts, part, C.byref(opts), bounds.ctypes.data,
                                          C.byref(sl), C.byref(h)))
        self.graph = DeviceGraph(h.value)
        self.bounds = bounds.astype(np.int64)
        self.slice = int(sl.value)
        self.n_global = full.n
        self.n_local = int(self.bounds[part + 1] - self.bounds[part])

    def init(self, exch) -> None:
        _check(lib().fpr_b200_part_init(self.graph._h, exch.data_ptr()))

    def sweep(self, engine: int, cfg: PageRankConfig, read, write, pair) -> None:
        c = cfg._c()
        _check(lib().fpr_b200_part_sweep(self.graph._h, engine, C.byref(c), read.data_ptr(),
                                         write.data_ptr(), pair.data_ptr()))

    def ranks(self) -> np.ndarray:
        out = np.empty(max(self.n_local, 1), np.float64)
        _check(lib().fpr_b200_part_ranks(self.graph._h, out.ctypes.data))
        return out[: self.n_local]

    def close(self):
        self.graph.close()


@dataclass
class PartResult:
    ranks: np.ndarray            # this part's rows
    errors: list = field(default_factory=list)
    l1_errors: list = field(default_factory=list)
    iterations: int = 0
    converged: bool = False
    iter_seconds: list = field(default_factory=list)


def _reduce_pairs(pairs: np.ndarray) -> tuple[float, float]:
    mx, sm = 0.0, 0.0
    for r in range(len(pairs) // 2):  # rank order: deterministic
        mx = max(mx, float(pairs[2 * r]))
        sm += float(pairs[2 * r + 1])
    return mx, sm


def solve_partitioned(local, exchange: TorchExchange, engine: int, cfg: PageRankConfig,
                      norm: int = NORM_LINF, device="cuda", want_ranks: bool = True) -> PartResult:
    """Run `engine` to convergence on this rank's part (one process per GPU).
    want_ranks=False leaves the part's ranks on the device (benchmarking)."""
    import torch

    if engine not in (ENGINE_EC, ENGINE_FUSED):
        raise ValueError("multi-GPU engines: EC or FUSED")
    P, S = exchange.world, local.slice
    a = torch.zeros(P * S, dtype=torch.float64, device=device)
    b = torch.zeros_like(a) if engine == ENGINE_EC else a
    pair = torch.zeros(2, dtype=torch.float64, device=device)
    local.init(a)
    exchange.allgather_slices(a, S)
    res = PartResult(np.empty(0))
    for it in range(int(cfg.max_iterations)):
        t0 = time.perf_counter()
        local.sweep(engine, cfg, a, b, pair)
        exchange.allgather_slices(b, S)
        pairs = exchange.allgather_pairs(pair).cpu().numpy()
        err, l1 = _reduce_pairs(pairs)
        res.iter_seconds.append(time.perf_counter() - t0)
        res.errors.append(err)
        res.l1_errors.append(l1)
        res.iterations = it + 1
        if engine == ENGINE_EC:
            a, b = b, a
        if (l1 if norm == NORM_L1 else err) <= cfg.threshold:
            break
    crit = res.l1_errors[-1] if norm == NORM_L1 else res.errors[-1]
    res.converged = crit <= cfg.threshold
    if want_ranks:
        res.ranks = local.ranks()
    return res


def solve_emulated(parts, engine: int, cfg: PageRankConfig, norm: int = NORM_LINF) -> PartResult:
    """All parts in one process on one GPU (EmulatedExchange): returns the
    concatenated global rank vector."""
    import torch

    P, S = len(parts), parts[0].slice
    ex = EmulatedExchange(P)
    A = [torch.zeros(P * S, dtype=torch.float64, device="cuda") for _ in range(P)]
    B = [torch.zeros_like(x) for x in A] if engine == ENGINE_EC else A
    pairs = [torch.zeros(2, dtype=torch.float64, device="cuda") for _ in range(P)]
    for r in range(P):
        parts[r].init(A[r])
    torch.cuda.synchronize()
    ex.allgather_slices_all(A, S)
    res = PartResult(np.empty(0))
    for it in range(int(cfg.max_iterations)):
        for r in range(P):
            parts[r].sweep(engine, cfg, A[r], B[r], pairs[r])
        torch.cuda.synchronize()
        ex.allgather_slices_all(B, S)
        err, l1 = _reduce_pairs(torch.cat(pairs).cpu().numpy())
        res.errors.append(err)
        res.l1_errors.append(l1)
        res.iterations = it + 1
        if engine == ENGINE_EC:
            A, B = B, A
        if (l1 if norm == NORM_L1 else err) <= cfg.threshold:
            break
    crit = res.l1_errors[-1] if norm == NORM_L1 else res.errors[-1]
    res.converged = crit <= cfg.threshold
    res.ranks = np.concatenate([p.ranks() for p in parts])
    return res
