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

Fused exchange (``fused_exchange=True``): instead of an all-gather after the
sweep, the sweep kernel's epilogue stores every finalized contribution into
each peer's replica as well (``fpr_b200_part_sweep_peers``; replicas mapped
with CUDA IPC, i.e. NVLink P2P stores through NVSwitch), so the exchange
overlaps the sweep row tile by row tile and only the 16-B residual pair
remains a collective -- which doubles as the inter-iteration barrier.
"""
from __future__ import annotations

import ctypes as C
import time
from dataclasses import dataclass, field

import numpy as np

from . import (B200Error, DeviceGraph, PageRankConfig, _check, _Config, _Options, _options, lib, ENGINE_EC,
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


_PINNED = {}


def _pinned_f64(count: int):
    """A reusable pinned host buffer of at least `count` doubles (pinned
    allocation costs milliseconds; a per-call one would dominate a D2H)."""
    import torch

    buf = _PINNED.get("f64")
    if buf is None or buf.numel() < count:
        buf = torch.empty(count, dtype=torch.float64, pin_memory=True)
        _PINNED["f64"] = buf
    return buf[:count]


# ------------------------------------------------------------------ local sweep
class B200Part:
    """This rank's part on its GPU, driven through the C ABI."""

    def __init__(self, full: DeviceGraph, nparts: int, part: int, device: int = 0, stream=None):
        # The exchange runs on torch's stream (NCCL / copies / .cpu()), so the
        # sweeps must too: default to torch's current stream, not a private one.
        if stream is None:
            from . import torch_stream_handle

            stream = torch_stream_handle()
        self.nparts, self.part = nparts, part
        self.device, self.stream = device, stream
        bounds = np.empty(nparts + 1, np.uint64)
        sl = C.c_uint64()
        h = C.c_void_p()
        L = lib()
        opts = _options(device=device, stream=stream)
        _check(L.fpr_b200_graph_partition(full._h, nparts, part, C.byref(opts), bounds.ctypes.data,
                                          C.byref(sl), C.byref(h)))
        self.graph = DeviceGraph(h.value)
        self.bounds = bounds.astype(np.int64)
        self.slice = int(sl.value)
        self.n_global = full.n
        self.n_local = int(self.bounds[part + 1] - self.bounds[part])

    @classmethod
    def from_view(cls, g, nparts: int, part: int, device: int = 0, stream=None) -> "B200Part":
        """This rank's part straight from a host fpr::Graph (pinned or pageable
        u64 arrays): only ~1/nparts of the graph is uploaded
        (fpr_b200_part_create); same bounds and slice as from a full DeviceGraph."""
        from . import _GraphView, _u64, torch_stream_handle

        if stream is None:
            stream = torch_stream_handle()
        ins, src, od = (a if isinstance(a, np.ndarray) and a.dtype == np.uint64 and a.flags.c_contiguous
                        else _u64(a) for a in (g.in_start, g.in_src, g.out_degree))
        v = _GraphView(g.n, g.m, ins.ctypes.data, src.ctypes.data if g.m else None, od.ctypes.data)
        bounds = np.empty(nparts + 1, np.uint64)
        sl = C.c_uint64()
        h = C.c_void_p()
        L = lib()
        _check(L.fpr_b200_part_create(C.byref(v), nparts, part, C.byref(_options(device=device, stream=stream)),
                                      bounds.ctypes.data, C.byref(sl), C.byref(h)))
        self = cls.__new__(cls)
        self.nparts, self.part = nparts, part
        self.device, self.stream = device, stream
        self.graph = DeviceGraph(h.value)
        self.bounds = bounds.astype(np.int64)
        self.slice = int(sl.value)
        self.n_global = g.n
        self.n_local = int(self.bounds[part + 1] - self.bounds[part])
        return self

    def init(self, exch) -> None:
        _check(lib().fpr_b200_part_init(self.graph._h, exch.data_ptr()))

    def sweep(self, engine: int, cfg: PageRankConfig, read, write, pair) -> None:
        c = cfg._c()
        _check(lib().fpr_b200_part_sweep(self.graph._h, engine, C.byref(c), read.data_ptr(),
                                         write.data_ptr(), pair.data_ptr()))

    def sweep_peers(self, engine: int, cfg: PageRankConfig, read, write, peer_ptrs, pair) -> None:
        """Fused exchange: the sweep also stores this part's slice straight into
        every other part's write vector (peer_ptrs[q], device addresses mapped
        into this process)."""
        c = cfg._c()
        arr = (C.c_void_p * len(peer_ptrs))(*peer_ptrs)
        L = lib()
        _check(L.fpr_b200_part_sweep_peers(self.graph._h, engine, C.byref(c), read.data_ptr(),
                                           write.data_ptr(), arr, len(peer_ptrs), pair.data_ptr()))

    def ranks(self, back: int = 0, out: np.ndarray | None = None) -> np.ndarray:
        """This part's ranks after the latest sweep, or (back=1) one sweep
        earlier.  `out` (n_local float64, ideally pinned) receives them
        directly; otherwise they go through a reusable pinned buffer (a
        pageable D2H of a large part runs at a fraction of the link rate)."""
        L = lib()
        fn = L.fpr_b200_part_ranks_prev if back else L.fpr_b200_part_ranks
        if out is not None:
            if out.dtype != np.float64 or not out.flags.c_contiguous or len(out) < self.n_local:
                raise ValueError("ranks: out must be a contiguous float64 array of n_local entries")
            _check(fn(self.graph._h, out.ctypes.data))
            return out[: self.n_local]
        pinned = _pinned_f64(max(self.n_local, 1))
        _check(fn(self.graph._h, pinned.data_ptr()))
        return pinned.numpy()[: self.n_local].copy()

    # -- device-side stop rule (fpr_b200_gate_*): no host round trip per iteration
    def gate_create(self, cap: int):
        """A gate (iteration count, stop flag, residual trace of `cap`
        iterations) in this part's device memory."""
        import torch

        nbytes = int(lib().fpr_b200_gate_bytes(cap))
        return {"buf": torch.zeros(nbytes, dtype=torch.uint8, device=f"cuda:{self.device}"), "cap": cap}

    def gate_init(self, gate) -> None:
        _check(lib().fpr_b200_gate_init(gate["buf"].data_ptr(), gate["cap"], self.device, self.stream))

    def set_gate(self, gate) -> None:
        """Bind (or with None unbind) the gate: sweeps are no-ops once it stopped."""
        _check(lib().fpr_b200_part_set_gate(self.graph._h, gate["buf"].data_ptr() if gate else None))

    def gate_update(self, gate, pairs, cfg: PageRankConfig, norm: int) -> None:
        """Enqueue the stop rule over the all-gathered pairs (2 x world doubles)."""
        world = pairs.numel() // 2
        base = pairs.data_ptr()
        arr = (C.c_void_p * world)(*[base + 16 * r for r in range(world)])
        c = cfg._c()
        _check(lib().fpr_b200_gate_update(gate["buf"].data_ptr(), arr, world, C.byref(c), norm, self.device,
                                          self.stream))

    def gate_read(self, gate, trace: bool = False):
        """(iterations, stopped, errors, l1_errors); waits for this part's stream."""
        it, st = C.c_uint64(), C.c_int()
        cap = gate["cap"] if trace else 0
        errs, l1s = np.zeros(cap), np.zeros(cap)
        _check(lib().fpr_b200_gate_read(gate["buf"].data_ptr(), self.device, self.stream, C.byref(it), C.byref(st),
                                        errs.ctypes.data if trace else None, l1s.ctypes.data if trace else None,
                                        cap))
        k = min(it.value, cap)
        return it.value, bool(st.value), errs[:k].tolist(), l1s[:k].tolist()

    def ranks_after(self, sweeps: int, out: np.ndarray | None = None) -> np.ndarray:
        """This part's ranks after sweep `sweeps` (later gated sweeps were no-ops)."""
        if out is None:
            pinned = _pinned_f64(max(self.n_local, 1))
            _check(lib().fpr_b200_part_ranks_after(self.graph._h, sweeps, pinned.data_ptr()))
            return pinned.numpy()[: self.n_local].copy()
        _check(lib().fpr_b200_part_ranks_after(self.graph._h, sweeps, out.ctypes.data))
        return out[: self.n_local]

    def close(self):
        self.graph.close()


# ------------------------------------------------------------ fused exchange
IPC_HANDLE_BYTES = 72  # FPR_B200_IPC_HANDLE_BYTES


def ipc_export(ptr: int) -> bytes:
    h = (C.c_char * IPC_HANDLE_BYTES)()
    L = lib()
    _check(L.fpr_b200_ipc_export(ptr, h))
    return bytes(h.raw)


def ipc_import(handle: bytes, device: int) -> int:
    out = C.c_void_p()
    L = lib()
    _check(L.fpr_b200_ipc_import(handle, device, C.byref(out)))
    return out.value


def ipc_close(ptr: int) -> None:
    L = lib()
    _check(L.fpr_b200_ipc_close(ptr))


class PeerReplicas:
    """Every part's exchange vectors mapped into this process, for the fused
    exchange: ptrs[k][q] = device address of part q's buffer k (its own buffer
    for q == rank, a CUDA-IPC mapping -- NVLink P2P on another GPU -- else).
    Handles travel over the process group (all_gather_object)."""

    def __init__(self, bufs, group=None, device: int = 0):
        import torch.distributed as dist

        self.rank = dist.get_rank(group)
        world = dist.get_world_size(group)
        mine = [ipc_export(b.data_ptr()) for b in bufs]
        everyone = [None] * world
        dist.all_gather_object(everyone, mine, group=group)
        self._opened = []
        self.ptrs = []
        for k, b in enumerate(bufs):
            row = []
            for q in range(world):
                if q == self.rank:
                    row.append(b.data_ptr())
                else:
                    ptr = ipc_import(everyone[q][k], device)
                    self._opened.append(ptr)
                    row.append(ptr)
            self.ptrs.append(row)

    def close(self):
        for ptr in self._opened:
            ipc_close(ptr)
        self._opened = []


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


class PartitionedSolver:
    """This rank's solver state, built once and reused across solves: the
    exchange vectors (two for EC's ping-pong, three when speculating; FUSED
    updates the first in place), the residual pairs and -- with
    fused_exchange -- the peers' replicas mapped through CUDA IPC.  If the
    replicas cannot be mapped (no P2P path), it falls back to the all-gather
    and says why in `fallback`.

    speculate=True (EC): sweep k+1 is enqueued before the host has read
    iteration k's residual, so the GPU never idles on the host round trip.
    Triple-buffered exchange vectors keep the extra sweep from touching
    anything iteration k needs; if k was the stopping iteration the part's
    ranks are read one sweep back (fpr_b200_part_ranks_prev), so results and
    the iteration count are the non-speculative ones.

    device_stop=True: the stop rule runs on the device (a gate,
    fpr_b200_gate_*).  Every iteration enqueues the sweep, the pair
    all-gather and the gate update without reading anything back; the host
    reads the gate once per `batch` iterations.  Sweeps issued after the
    stopping iteration are no-ops, and the ranks are those after the stopping
    sweep (fpr_b200_part_ranks_after), so the iteration count, trace and
    ranks equal the host-driven loop's."""

    def __init__(self, local, exchange: TorchExchange, device="cuda", fused_exchange: bool = False,
                 pairs_on_host: bool = False, speculate: bool = False, device_stop: bool = False,
                 batch: int = 8):
        import torch

        self.local, self.exchange, self.pairs_on_host = local, exchange, pairs_on_host
        self.speculate = speculate and not device_stop
        self.device_stop, self.batch, self._gate = device_stop, max(1, int(batch)), None
        P, S = exchange.world, local.slice
        self.bufs = [torch.zeros(P * S, dtype=torch.float64, device=device) for _ in range(3 if speculate else 2)]
        self.pairs = [torch.zeros(2, dtype=torch.float64, device=device) for _ in range(2)]
        self.reps, self.fallback = None, None
        if fused_exchange:
            dev = self.bufs[0].device.index or 0
            try:
                self.reps = PeerReplicas(self.bufs, exchange.group, dev)
            except B200Error as e:
                self.fallback = f"fused exchange unavailable ({e}); NCCL all-gather used"

    def rebind(self, local) -> None:
        """Reuse buffers and replicas for a re-created part of the same shape."""
        if local.slice != self.local.slice:
            raise ValueError("rebind: part slice differs")
        self.local = local

    @property
    def fused_exchange(self) -> bool:
        return self.reps is not None

    def _launch(self, j: int, engine: int, cfg: PageRankConfig):
        """Enqueue sweep j and its residual all-gather; returns a token for _wait."""
        import torch

        nb = len(self.bufs)
        ri, wi = (j % nb, (j + 1) % nb) if engine == ENGINE_EC else (0, 0)
        read, write = self.bufs[ri], self.bufs[wi]
        pair = self.pairs[j % 2]
        if self.reps is not None:
            # the sweep's epilogue stores into every peer replica (P2P)
            self.local.sweep_peers(engine, cfg, read, write, self.reps.ptrs[wi], pair)
        else:
            self.local.sweep(engine, cfg, read, write, pair)
            self.exchange.allgather_slices(write, self.local.slice)
        # the residual all-gather is also the barrier that keeps a fast rank
        # from writing a replica a slower peer is still reading
        out = self.exchange.allgather_pairs(pair.cpu() if self.pairs_on_host else pair)
        if out.is_cuda:
            host = torch.empty(out.shape, dtype=out.dtype, pin_memory=True)
            host.copy_(out, non_blocking=True)
            ev = torch.cuda.Event()
            ev.record()
            return host, ev
        return out, None

    @staticmethod
    def _wait(tok) -> np.ndarray:
        host, ev = tok
        if ev is not None:
            ev.synchronize()
        return host.numpy()

    def _solve_device_stop(self, engine: int, cfg: PageRankConfig, norm: int, want_ranks: bool,
                           ranks_out: np.ndarray | None) -> PartResult:
        local, exchange = self.local, self.exchange
        max_it = int(cfg.max_iterations)
        cap = min(max_it, 1 << 22)
        if self._gate is None or self._gate["cap"] < cap:
            self._gate = local.gate_create(cap)
        gate = self._gate
        local.init(self.bufs[0])
        exchange.allgather_slices(self.bufs[0], local.slice)
        local.gate_init(gate)
        local.set_gate(gate)
        res = PartResult(np.empty(0))
        t0 = time.perf_counter()
        try:
            issued, stopped = 0, False
            while not stopped and issued < max_it:
                for _ in range(min(self.batch, max_it - issued)):
                    nb = len(self.bufs)
                    ri, wi = (issued % nb, (issued + 1) % nb) if engine == ENGINE_EC else (0, 0)
                    read, write = self.bufs[ri], self.bufs[wi]
                    pair = self.pairs[issued % 2]
                    if self.reps is not None:
                        local.sweep_peers(engine, cfg, read, write, self.reps.ptrs[wi], pair)
                    else:
                        local.sweep(engine, cfg, read, write, pair)
                        exchange.allgather_slices(write, local.slice)
                    # the pair all-gather is the barrier; the gate update reads
                    # its result on the device, in rank order
                    if self.pairs_on_host:  # gloo groups (tests): through host memory
                        pairs = exchange.allgather_pairs(pair.cpu()).to(pair.device)
                    else:
                        pairs = exchange.allgather_pairs(pair)
                    local.gate_update(gate, pairs, cfg, norm)
                    issued += 1
                _, stopped, _, _ = local.gate_read(gate)
            it, stopped, errs, l1s = local.gate_read(gate, trace=True)
            if want_ranks:  # while bound: the sweeps past `it` were no-ops
                res.ranks = local.ranks_after(it, out=ranks_out)
        finally:
            local.set_gate(None)
        res.iterations, res.errors, res.l1_errors = it, errs, l1s
        res.iter_seconds = [(time.perf_counter() - t0) / max(it, 1)] * it
        crit = l1s[-1] if norm == NORM_L1 else errs[-1]
        res.converged = crit <= cfg.threshold
        return res

    def solve(self, engine: int, cfg: PageRankConfig, norm: int = NORM_LINF,
              want_ranks: bool = True, ranks_out: np.ndarray | None = None) -> PartResult:
        if engine not in (ENGINE_EC, ENGINE_FUSED):
            raise ValueError("multi-GPU engines: EC or FUSED")
        if self.device_stop:
            return self._solve_device_stop(engine, cfg, norm, want_ranks, ranks_out)
        spec = self.speculate and engine == ENGINE_EC
        local, exchange = self.local, self.exchange
        local.init(self.bufs[0])
        exchange.allgather_slices(self.bufs[0], local.slice)
        res = PartResult(np.empty(0))
        max_it = int(cfg.max_iterations)
        t0 = time.perf_counter()
        pend = self._launch(0, engine, cfg)
        ahead = None
        it = 0
        while True:
            nxt = self._launch(it + 1, engine, cfg) if spec and it + 1 < max_it else None
            err, l1 = _reduce_pairs(self._wait(pend))
            t1 = time.perf_counter()
            res.iter_seconds.append(t1 - t0)
            t0 = t1
            res.errors.append(err)
            res.l1_errors.append(l1)
            res.iterations = it + 1
            if (l1 if norm == NORM_L1 else err) <= cfg.threshold or it + 1 >= max_it:
                ahead = nxt
                break
            pend = nxt if nxt is not None else self._launch(it + 1, engine, cfg)
            it += 1
        if ahead is not None:
            self._wait(ahead)  # the extra sweep has finished everywhere before buffers are reused
        crit = res.l1_errors[-1] if norm == NORM_L1 else res.errors[-1]
        res.converged = crit <= cfg.threshold
        if want_ranks:
            res.ranks = local.ranks(back=1 if ahead is not None else 0, out=ranks_out)
        return res

    def close(self):
        if self.reps is not None:
            import torch

            torch.cuda.synchronize()
            self.exchange.dist.barrier(group=self.exchange.group)  # no peer still writes into ours
            self.reps.close()
            self.reps = None


def solve_partitioned(local, exchange: TorchExchange, engine: int, cfg: PageRankConfig,
                      norm: int = NORM_LINF, device="cuda", want_ranks: bool = True,
                      fused_exchange: bool = False, pairs_on_host: bool = False,
                      speculate: bool = False, device_stop: bool = False, batch: int = 8) -> PartResult:
    """Run `engine` to convergence on this rank's part (one process per GPU);
    a one-shot PartitionedSolver.  want_ranks=False leaves the part's ranks on
    the device (benchmarking).  fused_exchange=True replaces the per-iteration
    all-gather of contribution slices by the sweep's own P2P stores into the
    peers' replicas.  pairs_on_host moves the 16-B pair through host memory
    (gloo groups).  device_stop=True applies the stop rule on the device
    (PartitionedSolver)."""
    s = PartitionedSolver(local, exchange, device, fused_exchange, pairs_on_host, speculate, device_stop, batch)
    try:
        return s.solve(engine, cfg, norm, want_ranks)
    finally:
        s.close()


def solve_emulated(parts, engine: int, cfg: PageRankConfig, norm: int = NORM_LINF,
                   fused_exchange: bool = False) -> PartResult:
    """All parts in one process on one GPU (EmulatedExchange): returns the
    concatenated global rank vector.  fused_exchange=True has each part's
    sweep store its slice into the other parts' vectors (the P2P-store path
    with local pointers) instead of the copy exchange."""
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
            if fused_exchange:
                parts[r].sweep_peers(engine, cfg, A[r], B[r], [x.data_ptr() for x in B], pairs[r])
            else:
                parts[r].sweep(engine, cfg, A[r], B[r], pairs[r])
        torch.cuda.synchronize()
        if not fused_exchange:
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
