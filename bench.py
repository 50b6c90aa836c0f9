#!/usr/bin/env python
"""FusEd-PageRank B200 benchmark (driver contract: one JSON line on rank 0).

Workload (BASELINE.json configs[1], "config 2"): uniform G(n,m), n = 2^22,
2^26 draws of testutil::random_sparse(seed 2) semantics, normalised by
build_csr -> m = 67,108,723; fp64 ranks, d = 0.85, threshold 1e-10 on the
reference's L-inf delta.  The graph is generated ON THE DEVICE (K5 + K4,
bit-identical to the reference's CSR; untimed setup).

One step = one full ec_b200 solve to convergence (time-to-converge; 7
iterations).  value = GTEPS = m * iterations / step time, with the graph
resident in HBM.  e2e = the same metric through the reference-facing C-ABI
call fpr_b200_pagerank() on PINNED HOST u64 CSR arrays (fpr::Graph layout):
H2D + narrowing + partition + solve + D2H of ranks and error trace, all timed.

--impl reference: the reference's own CPU engine (oracle/_ref, compiled from
the unmodified headers), pagerank_ec_par with every host thread, one
iteration per step (a bounded sample of the same workload).
"""
from __future__ import annotations

import argparse
import ctypes as C
import json
import os
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

N_CFG2 = 1 << 22
DEG_CFG2 = 16
SEED_CFG2 = 2
THRESHOLD = 1e-10
DAMPING = 0.85
METRIC = "GTEPS/iter (EC PageRank to L-inf 1e-10, config 2)"
WORKLOAD = "config2: uniform G(n=4194304, 2^26 draws, seed 2) -> build_csr, EC to L-inf 1e-10"


def algorithmic_bytes(n: int, m: int) -> int:
    """Per iteration: 12 B/edge (int32 in_src + fp64 contrib gather) +
    36 B/vertex (int64 row_ptr, pr read+write, int32 outdeg, contrib write)."""
    return 12 * m + 36 * n


def ncu_traffic(key: str, launches_per_step: int) -> float | None:
    """DRAM read+write bytes per solve launch from the committed ncu capture."""
    try:
        with open(os.path.join(ROOT, "profiles", "traffic.json")) as f:
            return float(json.load(f)[key]["dram_bytes_per_launch"])
    except Exception:
        return None


def peaks() -> tuple[float, str]:
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            return float(json.load(f)["hbm_gbs"]), "measured"
    except Exception:
        return 6650.0, "fallback"


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled every 20 ms during the
    timed region (one `nvidia-smi -lms` process, started before, stopped after)."""

    Q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")

    def __init__(self, device: int):
        self.device = device
        self.rows: list[list[str]] = []
        self.proc = None

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.device), f"--query-gpu={self.Q}",
                                          "--format=csv,noheader,nounits", "-lms", "20"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            time.sleep(0.3)  # first sample lands before the timed region starts
        except Exception:
            self.proc = None
        return self

    def __exit__(self, *a):
        if self.proc is None:
            return
        time.sleep(0.05)
        self.proc.terminate()
        try:
            out, _ = self.proc.communicate(timeout=5)
        except Exception:
            self.proc.kill()
            out = ""
        self.rows = [[x.strip() for x in line.split(",")] for line in out.splitlines() if line.strip()]

    def summary(self) -> dict:
        if not self.rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"], "samples": 0}
        sm = [float(r[0]) for r in self.rows if r[0].replace(".", "").isdigit()]
        mx = [float(r[1]) for r in self.rows if len(r) > 1 and r[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in self.rows for i in range(4)
                          if len(r) > 2 + i and r[2 + i].lower() == "active"})
        return {"sm_mhz": float(np.median(sm)) if sm else None,
                "sm_max_mhz": max(mx) if mx else None, "reasons": reasons, "samples": len(self.rows)}


def dist_env():
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return ws, rank, local


def reference_graph(ref):
    """Config-2 graph built by the reference's own functions."""
    n, s, d = ref.random_sparse(N_CFG2, DEG_CFG2, SEED_CFG2)
    return ref.build_csr(n, s, d)


def run_reference(args) -> None:
    ws, rank, _ = dist_env()
    if rank != 0:
        return
    from oracle import Oracle, load_reference

    ref = load_reference()
    threads = os.cpu_count() or 1
    if ref is not None:
        kind = "reference"
        g = reference_graph(ref)
        h = ref.graph_handle(g)
        one = lambda: ref.run(g, "ec_par", DAMPING, THRESHOLD, 1, threads, handle=h).seconds  # noqa: E731
        engine = "fpr::pagerank_ec_par (oracle/_ref, unmodified reference headers)"
    else:  # reference not compiled on this box: the C restatement (single thread)
        kind = "port"
        o = Oracle()
        n, s, d = o.random_sparse(N_CFG2, DEG_CFG2, SEED_CFG2)
        g = o.build_csr(n, s, d)
        threads = 1

        def one():
            t0 = time.perf_counter()
            o.pagerank_ec(g, DAMPING, THRESHOLD, 1)
            return time.perf_counter() - t0
        engine = "oracle/fpr_oracle.c fo_pagerank_ec (C restatement, 1 thread)"
    for _ in range(args.warmup):
        one()
    secs = [one() for _ in range(args.steps)]
    t = float(sum(secs))
    gteps = g.m * args.steps / t / 1e9
    line = {"metric": METRIC, "value": gteps, "unit": "GTEPS",
            "impl": "reference", "n_gpus": ws, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": 1e3 * t / args.steps, "higher_is_better": True, "scaling": "strong",
            "vs_baseline": None, "dtype": "f64", "data": "synthetic (random_sparse seed 2)",
            "config": {"workload": WORKLOAD, "n": g.n, "m": g.m, "step": "1 EC iteration",
                       "engine": engine},
            "cpu_baseline": {"value": gteps, "unit": "GTEPS", "cores": threads, "kind": kind,
                             "sample": f"{args.steps} single-iteration ec_par calls on config 2"},
            "e2e": {"value": gteps, "unit": "GTEPS", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    if ref is not None:
        ref.destroy(h)
    print(json.dumps(line), flush=True)


def cpu_baseline_leg(g_host, gpu_ranks=None, gpu_iters=None) -> dict:
    """Rank 0, N=1: the reference's ec_par, all host threads, one full solve.
    Its converged vector doubles as a live parity check of the GPU result."""
    from oracle import Graph as OGraph
    from oracle import Oracle, load_reference

    ref = load_reference()
    og = OGraph(g_host.n, g_host.m, g_host.in_start, g_host.in_src, g_host.out_degree)
    if ref is not None:
        threads = os.cpu_count() or 1
        h = ref.graph_handle(og)
        try:
            r = ref.run(og, "ec_par", DAMPING, THRESHOLD, 10000, threads, handle=h)
        finally:
            ref.destroy(h)
        out = {"value": og.m * r.iterations / r.seconds / 1e9, "unit": "GTEPS", "cores": threads,
               "kind": "reference", "iterations": r.iterations, "seconds": r.seconds,
               "sample": "1 full pagerank_ec_par solve of config 2 (oracle/_ref, -O3, T=nproc)"}
        if gpu_ranks is not None:
            out["parity"] = {"ec_b200_vs_reference_max_rel": float(np.max(np.abs(gpu_ranks - r.ranks) / r.ranks)),
                             "iterations_equal": bool(gpu_iters == r.iterations), "tolerance": 1e-12}
        return out
    o = Oracle()
    t0 = time.perf_counter()
    r = o.pagerank_ec(og, DAMPING, THRESHOLD, 2)
    dt = time.perf_counter() - t0
    return {"value": og.m * r.iterations / dt / 1e9, "unit": "GTEPS", "cores": 1, "kind": "port",
            "iterations": r.iterations, "seconds": dt,
            "sample": "2 EC iterations of config 2 with the C restatement (1 thread)"}


def render_fixed(src, dst, width=7) -> np.ndarray:
    """Bench input for the ingest leg: one "%0{width}d %0{width}d\\n" line per
    edge (leading zeros are valid from_chars tokens, edge_list.hpp:25-30)."""
    out = np.empty((len(src), 2 * width + 2), np.uint8)
    for col, ids in ((0, src), (width + 1, dst)):
        v = np.asarray(ids, dtype=np.uint64).copy()
        for k in range(width - 1, -1, -1):
            out[:, col + k] = (v % np.uint64(10)).astype(np.uint8) + 48
            v //= np.uint64(10)
    out[:, width] = 32
    out[:, 2 * width + 1] = 10
    return out.reshape(-1)


def ingest_leg(fb, g, device) -> dict:
    """§8(f) edge-list ingest: config 2's edges as text -> resident device CSR
    through fpr_b200_graph_from_edge_list (pinned host text, H2D inside the
    timed call), against the reference's parse_edge_list + build_csr on a
    1/64 sample (single thread: the reference parser is sequential)."""
    import torch

    dst = np.repeat(np.arange(g.n, dtype=np.uint64), np.diff(g.in_start.astype(np.int64)))
    text = render_fixed(g.in_src, dst)
    pinned = torch.empty(len(text), dtype=torch.uint8, pin_memory=True)
    pinned.numpy()[:] = text
    buf = pinned.numpy()
    fb.DeviceGraph.from_edge_list(buf, device=device).close()  # warm-up
    times = []
    for _ in range(3):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        d = fb.DeviceGraph.from_edge_list(buf, device=device)
        torch.cuda.synchronize()
        times.append(time.perf_counter() - t0)
        assert d.m == g.m
        d.close()
    dt = float(np.median(times))
    out = {"workload": f"config-2 edges as '%07d %07d\\n' text ({len(text) / 1e9:.2f} GB, {g.m} lines)",
           "api": "fpr_b200_graph_from_edge_list (pinned host text -> resident CSR; H2D timed)",
           "ms": dt * 1e3, "medges_per_s": g.m / dt / 1e6, "text_gb_per_s": len(text) / dt / 1e9,
           "h2d_bytes": int(len(text))}
    try:
        from oracle import load_reference

        ref = load_reference()
        if ref is not None:
            sample = text[: (len(text) // 64 // 16) * 16].tobytes()
            t0 = time.perf_counter()
            p = ref.parse_edge_list(sample)
            ref.build_csr(p.n, p.edges[:, 0], p.edges[:, 1])
            rdt = time.perf_counter() - t0
            out["reference"] = {"medges_per_s": len(p.edges) / rdt / 1e6, "kind": "reference", "cores": 1,
                                "sample": f"parse_edge_list + build_csr of the first {len(p.edges)} lines"}
    except Exception as ex:  # reference arm is informative only
        out["reference"] = {"unavailable": str(ex)}
    return out


def large_configs_leg(fb, device, which=("3", "4", "5", "5r")) -> dict:
    """BASELINE configs 3-5 on one GPU, generated on the device (untimed):
    EC and FusEd time-to-converge at L-inf 1e-10, ms per sweep, GTEPS and
    the HBM-roofline fraction (12 m + 36 n bytes per sweep); on configs 4/5
    also the propagation-blocked engines (FPR_B200_OPT_PB): EC, and the
    lockstep FusEd schedule on PB sweeps (auto wave count).  Not the
    headline metric; reported beside it.  Solve times are CUDA-event times
    of the solve launches (resident graph)."""
    cfg = fb.PageRankConfig(damping=DAMPING, threshold=THRESHOLD)
    peak, _ = peaks()
    out = {}

    def record(dg, r):
        ms_it = r.solve_ms / r.trace.iterations
        return {"iterations": r.trace.iterations, "converged": bool(r.trace.converged),
                "time_to_converge_ms": r.solve_ms, "ms_per_sweep": ms_it, "gteps": dg.m / ms_it / 1e6,
                "roofline_frac": algorithmic_bytes(dg.n, dg.m) / (ms_it * 1e-3) / 1e9 / peak}

    for c in which:
        if c == "3":
            dg = fb.DeviceGraph.generate_rmat(fb.RmatParams(24, 16, seed=3), relabel_bfs=True, device=device)
            name = "config3: RMAT s24 ef16 seed 3, BFS crawl-order relabel"
        elif c == "4":
            dg = fb.DeviceGraph.generate_chunglu(1 << 26, 1_200_000_000, seed=4, device=device)
            name = "config4: Chung-Lu n=2^26, 1.2e9 draws, alpha 2.1, seed 4, random order"
        else:
            dg = fb.DeviceGraph.generate_rmat(fb.RmatParams(28, 16, seed=5), device=device,
                                              reorder=c.endswith("r"))
            name = "config5: RMAT s28 ef16 seed 5" + (" + FPR_B200_OPT_REORDER" if c.endswith("r") else "")
        with dg:
            rec = {"workload": name, "n": dg.n, "m": dg.m}
            for eng, tag in ((fb.ENGINE_EC, "ec"), (fb.ENGINE_FUSED, "fused")):
                rec[tag] = record(dg, dg.run(eng, cfg, copy_ranks=False, copy_trace=False))
            out["config" + c] = rec
        if c != "3":
            # FPR_B200_OPT_PB (propagation-blocked EC) on a
            # second handle; its one-time layout build is outside solve_ms
            if c == "4":
                dg = fb.DeviceGraph.generate_chunglu(1 << 26, 1_200_000_000, seed=4, device=device, pb=True)
            else:
                dg = fb.DeviceGraph.generate_rmat(fb.RmatParams(28, 16, seed=5), device=device,
                                                  reorder=c.endswith("r"), pb=True)
            with dg:
                one = fb.PageRankConfig(damping=DAMPING, threshold=THRESHOLD, max_iterations=1)
                for eng, tag in ((fb.ENGINE_EC, "ec_pb"), (fb.ENGINE_FUSED_LOCKSTEP, "lockstep_pb")):
                    first = dg.run(eng, one, copy_ranks=False, copy_trace=False)  # builds the layout / wave plan
                    rec[tag] = record(dg, dg.run(eng, cfg, copy_ranks=False, copy_trace=False))
                    # one-time device setup on this handle (EC: the PB layout; lockstep: its wave plan)
                    rec[tag]["setup_ms_first_run"] = first.setup_ms
                    # the PB sweep's own streamed bytes: 22 B per edge
                    # (source, value written and read back, row offset) + 36 B per vertex
                    ms_it = rec[tag]["ms_per_sweep"]
                    rec[tag]["pb_stream_bytes_frac"] = (22 * dg.m + 36 * dg.n) / (ms_it * 1e-3) / 1e9 / peak
                rec["lockstep_pb"]["waves"] = len(dg.wave_starts()) - 1
    return out


def build_csr_leg(fb, g, device) -> dict:
    """Graph loading (§8(a) a12): fpr::build_csr(EdgeSet) of config 2's edges
    (pinned host u64 src/dst, H2D + narrowing + device sort/dedup/scan timed)
    through fpr_b200_graph_from_edges, against the reference's build_csr on a
    1/16 sample of the same edges (single thread, as the reference runs)."""
    import torch

    dst = np.repeat(np.arange(g.n, dtype=np.uint64), np.diff(g.in_start.astype(np.int64)))
    ts = torch.empty(g.m, dtype=torch.int64, pin_memory=True)
    td = torch.empty(g.m, dtype=torch.int64, pin_memory=True)
    s, d = ts.numpy().view(np.uint64), td.numpy().view(np.uint64)
    s[:] = g.in_src
    d[:] = dst
    fb.DeviceGraph.from_edges(g.n, s, d, device=device).close()  # warm-up
    times = []
    for _ in range(3):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        dg = fb.DeviceGraph.from_edges(g.n, s, d, device=device)
        torch.cuda.synchronize()
        times.append(time.perf_counter() - t0)
        assert dg.m == g.m
        dg.close()
    dt = float(np.median(times))
    out = {"workload": f"config-2 edges as an EdgeSet (n={g.n}, {g.m} edges)",
           "api": "fpr_b200_graph_from_edges (pinned host u64 src/dst -> resident CSR + partition)",
           "ms": dt * 1e3, "medges_per_s": g.m / dt / 1e6, "h2d_bytes": int(16 * g.m)}
    try:
        from oracle import load_reference

        ref = load_reference()
        if ref is not None:
            k = g.m // 16
            rng = np.random.default_rng(0)
            pick = np.sort(rng.choice(g.m, size=k, replace=False))
            t0 = time.perf_counter()
            ref.build_csr(g.n, s[pick].copy(), d[pick].copy())
            rdt = time.perf_counter() - t0
            out["reference"] = {"medges_per_s": k / rdt / 1e6, "kind": "reference", "cores": 1,
                                "sample": f"build_csr of a random 1/16 of the edges ({k}), n = {g.n}"}
    except Exception as ex:
        out["reference"] = {"unavailable": str(ex)}
    return out


def main() -> None:
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=100)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-ingest", action="store_true")
    ap.add_argument("--no-large", action="store_true", help="skip configs 3-5 (about 1 min)")
    ap.add_argument("--copy-exchange", action="store_true",
                    help="N>1: NCCL all-gather of slices instead of the fused P2P-store exchange")
    ap.add_argument("--partitioned", action="store_true",
                    help="use the multi-GPU partitioned path even at N=1 (NCCL world of 1)")
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3)
    if args.impl == "reference":
        run_reference(args)
        return

    import torch

    import paper_2203_09284_b200 as fb

    ws, rank, local = dist_env()
    torch.cuda.set_device(local)
    dist = None
    if ws > 1 or args.partitioned:
        import os as _os

        import torch.distributed as dist

        if ws == 1:
            _os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
            _os.environ.setdefault("MASTER_PORT", "29531")
            _os.environ.setdefault("RANK", "0")
            _os.environ.setdefault("WORLD_SIZE", "1")
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        run_multi(args, fb, dist, ws, rank, local)
        dist.destroy_process_group()
        return
    stream = torch.cuda.current_stream()
    sptr = fb.torch_stream_handle()

    dg = fb.DeviceGraph.generate_uniform(N_CFG2, DEG_CFG2, SEED_CFG2, device=local, stream=sptr)
    n, m = dg.n, dg.m
    cfg = fb.PageRankConfig(damping=DAMPING, threshold=THRESHOLD)

    def step():
        return dg.run(fb.ENGINE_EC, cfg, copy_ranks=False, copy_trace=False)

    for _ in range(args.warmup):
        r = step()
    iters = r.trace.iterations
    launches_per_step = r.kernel_launches

    def barrier():
        if dist is not None:
            dist.barrier()
        torch.cuda.synchronize()

    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    kernel_ms = []
    with ClockSampler(local) as clk:
        barrier()
        ev0.record(stream)
        for _ in range(args.steps):
            r = step()
            kernel_ms.append(r.solve_ms)
            assert r.trace.iterations == iters
        ev1.record(stream)
        barrier()
    ms = ev0.elapsed_time(ev1)
    if dist is not None:
        t = torch.tensor([ms], device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())
    ms_step = ms / args.steps
    value = ws * m * iters / (ms_step * 1e-3) / 1e9
    kms = float(np.mean(kernel_ms))
    peak, peak_kind = peaks()
    achieved = algorithmic_bytes(n, m) * iters / (kms * 1e-3) / 1e9

    # Per-iteration device times of the persistent kernel (globaltimer).
    tr = dg.run(fb.ENGINE_EC, cfg, copy_ranks=False, copy_trace=True)
    it_us = (tr.trace.iter_ns.astype(np.float64) / 1e3).tolist()

    # FusEd (block-async) on the same resident graph.
    fused = {}
    fr = [dg.run(fb.ENGINE_FUSED, cfg, copy_ranks=False, copy_trace=False) for _ in range(max(3, args.steps // 4))]
    fused = {"engine": "fused_b200", "iterations": fr[-1].trace.iterations,
             "roofline_frac": algorithmic_bytes(n, m) * fr[-1].trace.iterations
             / (float(np.mean([x.solve_ms for x in fr])) * 1e-3) / 1e9 / peaks()[0],
             "iterations_min_max": [min(x.trace.iterations for x in fr), max(x.trace.iterations for x in fr)],
             "ms_per_solve": float(np.mean([x.solve_ms for x in fr])),
             "gteps": float(np.mean([m * x.trace.iterations / x.solve_ms / 1e6 for x in fr]))}
    lr = dg.run(fb.ENGINE_FUSED_LOCKSTEP, cfg, copy_ranks=False, copy_trace=False)
    fused["lockstep"] = {"iterations": lr.trace.iterations, "ms_per_solve": lr.solve_ms,
                         "waves": int(len(dg.wave_starts()) - 1)}

    # BASELINE.json words the stop rule as an L1 delta; the reference stops on
    # L-inf (the headline).  Same graph, L1 rule, reported beside it.
    l1_stop = {}
    with fb.DeviceGraph.generate_uniform(N_CFG2, DEG_CFG2, SEED_CFG2, device=local, stream=sptr,
                                         norm=fb.NORM_L1) as dl1:
        for eng, tag in ((fb.ENGINE_EC, "ec"), (fb.ENGINE_FUSED_LOCKSTEP, "fused_lockstep"),
                         (fb.ENGINE_FUSED, "fused")):
            dl1.run(eng, cfg, copy_ranks=False, copy_trace=False)
            r1 = dl1.run(eng, cfg, copy_ranks=False, copy_trace=False)
            l1_stop[tag] = {"iterations": r1.trace.iterations, "time_to_converge_ms": r1.solve_ms,
                            "converged": bool(r1.trace.converged)}
    g_host = None
    e2e = None
    if not args.no_e2e:
        g_host = dg.download()
        e2e = e2e_leg(fb, g_host, local, args, iters)
    ingest = None
    if rank == 0 and ws == 1 and not args.no_ingest:
        if g_host is None:
            g_host = dg.download()
        ingest = ingest_leg(fb, g_host, local)
    csr = None
    if rank == 0 and ws == 1 and not args.no_ingest:
        if g_host is None:
            g_host = dg.download()
        csr = build_csr_leg(fb, g_host, local)
    large = None
    if rank == 0 and ws == 1 and not args.no_large:
        large = large_configs_leg(fb, local)
    cpu = None
    if rank == 0 and ws == 1 and not args.no_cpu_baseline:
        if g_host is None:
            g_host = dg.download()
        final = dg.run(fb.ENGINE_EC, cfg, copy_ranks=True, copy_trace=False)
        cpu = cpu_baseline_leg(g_host, final.ranks.values, final.trace.iterations)

    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": "GTEPS",
            "n_gpus": ws, "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms_step,
            # config 2 at every N: total work fixed (N > 1 partitions it, run_multi)
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic (device-generated, bit-identical to reference random_sparse+build_csr)",
            "config": {"workload": WORKLOAD, "n": n, "m": m, "iterations": iters, "threshold": THRESHOLD,
                       "norm": "linf", "step": "1 full EC solve (time-to-converge)",
                       "parallelism": "single-gpu",
                       "l2": "inputs larger than L2 (in_src 268 MB + contrib 33.5 MB + row_ptr 33.5 MB); no flush"},
            "time_to_converge_ms": ms_step,
            "iteration_us": it_us,
            "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                         "frac": achieved / peak, "traffic": ncu_traffic("config2_ec", 1), "peak_kind": peak_kind,
                         "traffic_unit": "bytes per launch (ncu dram__bytes_read+write, profiles/traffic.json)",
                         # the random-fetch ceiling measured by bench_micro/gather_bench.cu (an
                         # L2-side request limit): the kernel's real bound on config 2
                         "gather_ceiling_gteps": 270.0,
                         "gather_ceiling_frac": m * iters / (kms * 1e-3) / 1e9 / 270.0,
                         "kernel": "solve_kernel<false> (persistent EC, all iterations)",
                         "kernel_ms": kms,
                         "algorithmic_bytes_per_launch": algorithmic_bytes(n, m) * iters},
            "fused": fused,
            "l1_stop_rule": l1_stop,
            "cpu_baseline": cpu,
            "e2e": e2e,
            "ingest": ingest,
            "build_csr": csr,
            "configs_3_5": large,
            "gpu_launches": int(launches_per_step * args.steps),
            "clocks": clk.summary(),
        }
        print(json.dumps(line), flush=True)
    dg.close()
    if dist is not None:
        dist.destroy_process_group()


def run_multi(args, fb, dist, ws, rank, local) -> None:
    """N GPUs: destination-range partition of config 2 (strong scaling), one
    NCCL all-gather of contribution slices + one residual all-gather per
    iteration (paper_2203_09284_b200/dist.py)."""
    import torch

    from paper_2203_09284_b200.dist import B200Part, PartitionedSolver, TorchExchange

    sptr = fb.torch_stream_handle()
    full = fb.DeviceGraph.generate_uniform(N_CFG2, DEG_CFG2, SEED_CFG2, device=local, stream=sptr)
    n, m = full.n, full.m
    part = B200Part(full, ws, rank, device=local, stream=sptr)
    full.close()
    ex = TorchExchange()
    cfg = fb.PageRankConfig(damping=DAMPING, threshold=THRESHOLD)
    dev = f"cuda:{local}"
    # fused exchange: the sweep stores its slice into the peers' replicas
    # (CUDA IPC / NVLink P2P); NCCL carries only the 16-B residual pair
    # Speculation costs one extra sweep per solve and saves a host round trip
    # per iteration: a win once the sweep is short (N > 1), a loss at N = 1.
    solver = PartitionedSolver(part, ex, device=dev, fused_exchange=not args.copy_exchange and ws > 1,
                               speculate=ws > 1)
    for _ in range(args.warmup):
        r = solver.solve(fb.ENGINE_EC, cfg, want_ranks=False)
    iters = r.iterations

    def barrier():
        dist.barrier()
        torch.cuda.synchronize()

    stream = torch.cuda.current_stream()
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(local) as clk:
        barrier()
        ev0.record(stream)
        for _ in range(args.steps):
            r = solver.solve(fb.ENGINE_EC, cfg, want_ranks=False)
            assert r.iterations == iters
        ev1.record(stream)
        barrier()
    t = torch.tensor([ev0.elapsed_time(ev1)], device=dev)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    ms_step = float(t.item()) / args.steps
    fr = solver.solve(fb.ENGINE_FUSED, cfg, want_ranks=False)
    e2e = None
    if not args.no_e2e:
        e2e = e2e_multi(args, fb, dist, solver, cfg, dev, local, iters)
    exchange = ("fused: sweep epilogue P2P-stores each slice into the peers' replicas (CUDA IPC over NVLink); "
                "NCCL all-gather of the 16-B residual pair" if solver.fused_exchange else
                "NCCL all-gather of contribution slices + residual pair")
    if rank == 0:
        line = {
            "metric": METRIC,
            "value": m * iters / (ms_step * 1e-3) / 1e9, "unit": "GTEPS", "n_gpus": ws,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms_step,
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic (device-generated, bit-identical to reference random_sparse+build_csr)",
            "config": {"workload": WORKLOAD, "n": n, "m": m, "iterations": iters, "threshold": THRESHOLD,
                       "norm": "linf", "step": "1 full EC solve (time-to-converge)",
                       "parallelism": f"dst-range partition x{ws}", "exchange": exchange,
                       "host_loop": ("speculative: sweep k+1 enqueued before iteration k's residual is read"
                                     if ws > 1 else "synchronous"),
                       "exchange_fallback": solver.fallback,
                       "slice": part.slice, "l2": "inputs larger than L2; no flush"},
            "time_to_converge_ms": ms_step,
            "fused": {"engine": "fused_b200", "iterations": fr.iterations},
            "roofline": None, "cpu_baseline": None, "e2e": e2e,
            "gpu_launches": int(args.steps * iters), "clocks": clk.summary(),
        }
        print(json.dumps(line), flush=True)
    solver.close()
    part.close()


def e2e_multi(args, fb, dist, solver, cfg, dev, local, iters) -> dict:
    """N GPUs end to end through the public API: every rank uploads only its
    own rows of the pinned host CSR (fpr_b200_part_create), solves with the
    partitioned driver and downloads its rank slice.  Max over ranks."""
    import torch

    from paper_2203_09284_b200.dist import B200Part

    g = None
    with fb.DeviceGraph.generate_uniform(N_CFG2, DEG_CFG2, SEED_CFG2, device=local,
                                         stream=fb.torch_stream_handle()) as dg:
        g = dg.download()

    def pinned(a):
        t = torch.empty(a.shape, dtype=torch.int64, pin_memory=True)
        v = t.numpy().view(np.uint64)
        v[:] = a
        return t, v

    keep = [pinned(g.in_start), pinned(g.in_src), pinned(g.out_degree)]
    hg = fb.Graph(g.n, g.m, keep[0][1], keep[1][1], keep[2][1])
    ws, rank = dist.get_world_size(), dist.get_rank()

    ranks_host = torch.empty(g.n, dtype=torch.float64, pin_memory=True).numpy()  # >= any part's rows

    def call():
        # each rank uploads only its own rows (fpr_b200_part_create)
        p = B200Part.from_view(hg, ws, rank, device=local, stream=fb.torch_stream_handle())
        old = solver.local
        solver.rebind(p)  # exchange buffers / peer replicas are persistent state
        r = solver.solve(fb.ENGINE_EC, cfg, want_ranks=True, ranks_out=ranks_host)
        solver.rebind(old)
        p.close()
        return r

    call()
    steps = max(3, min(args.steps, 10))
    dist.barrier()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(steps):
        r = call()
    torch.cuda.synchronize()
    t = torch.tensor([(time.perf_counter() - t0) / steps], device=dev)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    dt = float(t.item())
    h2d = 8 * (g.n + 1) + 8 * g.m + 8 * g.n
    d2h = 8 * len(r.ranks) + 16 * ws * r.iterations
    return {"value": g.m * r.iterations / dt / 1e9, "unit": "GTEPS", "h2d_bytes_per_step": h2d,
            "d2h_bytes_per_step": d2h, "ms_per_step": dt * 1e3, "steps": steps,
            "api": "fpr_b200_part_create + fpr_b200_part_* (pinned host u64 CSR, each rank uploads its rows)"}


def e2e_leg(fb, g, device, args, iters) -> dict:
    """fpr_b200_pagerank() on pinned host fpr::Graph arrays; H2D + solve + D2H timed."""
    import torch

    def pinned(a):
        t = torch.empty(a.shape, dtype=torch.int64, pin_memory=True)
        v = t.numpy().view(np.uint64)
        v[:] = a
        return t, v

    keep = [pinned(g.in_start), pinned(g.in_src), pinned(g.out_degree)]
    ins, src, od = (k[1] for k in keep)
    ranks_t = torch.empty(g.n, dtype=torch.float64, pin_memory=True)
    errs_t = torch.empty(10000, dtype=torch.float64, pin_memory=True)
    view = fb._GraphView(g.n, g.m, ins.ctypes.data, src.ctypes.data, od.ctypes.data)
    cfg = fb.PageRankConfig(damping=DAMPING, threshold=THRESHOLD)._c()
    opts = fb._options(device=device, stream=fb.torch_stream_handle())
    res = fb._Result()
    L = fb.lib()

    def call():
        fb._check(L.fpr_b200_pagerank(C.byref(view), fb.ENGINE_EC, C.byref(cfg), C.byref(opts),
                                      ranks_t.data_ptr(), errs_t.data_ptr(), 10000, C.byref(res)))

    for _ in range(2):
        call()
    steps = max(3, min(args.steps, 20))
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(steps):
        call()
    dt = (time.perf_counter() - t0) / steps
    assert res.iterations == iters
    h2d = 8 * (g.n + 1) + 8 * g.m + 8 * g.n
    d2h = 8 * g.n + 8 * int(res.iterations)
    return {"value": g.m * res.iterations / dt / 1e9, "unit": "GTEPS", "h2d_bytes_per_step": h2d,
            "d2h_bytes_per_step": d2h, "ms_per_step": dt * 1e3, "steps": steps,
            "api": "fpr_b200_pagerank (C ABI, pinned host u64 CSR)"}


if __name__ == "__main__":
    main()
