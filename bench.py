#!/usr/bin/env python
"""FusEd-PageRank B200 benchmark (driver contract: one JSON line on rank 0).

Headline workload (BASELINE.json configs[4], "config 5", the largest graph
that fits one GPU): R-MAT scale 28, edge factor 16, a/b/c/d = .57/.19/.19/.05,
seed 5, normalised by build_csr -> n = 2^28, m = 4,259,432,546; fp64 ranks,
d = 0.85, threshold 1e-10 on the reference's L-inf delta.  The graph is
generated ON THE DEVICE (K5 + K4, bit-identical to the reference's
generate_rmat + build_csr by construction; pinned by digests up to scale 24).

One step = one full ec_b200 solve to convergence on the sweep the library
picks by default (propagation-blocked on this graph) -- the
time-to-converge, 54 iterations.  value = GTEPS/iter = m * iterations / step
time, graph resident in HBM (inputs far larger than L2: no flush needed).
e2e = the same metric through the reference-facing C-ABI call
fpr_b200_pagerank() on PINNED HOST u64 CSR arrays (the fpr::Graph layout, 38
GB): H2D + narrowing + the one-time sweep layout + solve + D2H of ranks and
error trace, all timed.

--impl reference: the reference's own CPU engine (oracle/_ref, compiled from
the unmodified headers), fpr::pagerank_ec_par with every host thread, on the
same config-5 graph.  A full reference solve takes ~23 minutes on the GPU
box's 16 cores (54 iterations x ~25 s), so its step is a bounded sample: one
pagerank_ec_par call of 3 iterations (per-iteration cost, GTEPS/iter);
setup (graph hand-off + the reference's build_layout, ~3 min) is untimed.
"""
from __future__ import annotations

import argparse
import ctypes as C
import json
import os
import subprocess
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

THRESHOLD = 1e-10
DAMPING = 0.85
METRIC = "GTEPS/iter (EC PageRank to L-inf 1e-10, time-to-converge)"

WORKLOADS = {
    "5": "config5: RMAT s28 ef16 (a,b,c,d)=(.57,.19,.19,.05) seed 5 -> build_csr, EC to L-inf 1e-10",
    "2": "config2: uniform G(n=4194304, 2^26 draws, seed 2) -> build_csr, EC to L-inf 1e-10",
    "1": "config1: RMAT s16 ef16 (a,b,c,d)=(.57,.19,.19,.05) seed 1 -> build_csr, EC to L-inf 1e-10",
}
REF_SAMPLE_ITERS = 3  # --impl reference: iterations in its one timed pagerank_ec_par call


def make_graph(fb, config: str, device, stream=None, **kw):
    if config == "1":
        return fb.DeviceGraph.generate_rmat(fb.RmatParams(16, 16, seed=1), device=device, stream=stream, **kw)
    if config == "2":
        return fb.DeviceGraph.generate_uniform(1 << 22, 16, 2, device=device, stream=stream, **kw)
    if config == "3":
        return fb.DeviceGraph.generate_rmat(fb.RmatParams(24, 16, seed=3), relabel_bfs=True, device=device,
                                            stream=stream, **kw)
    if config == "4":
        return fb.DeviceGraph.generate_chunglu(1 << 26, 1_200_000_000, seed=4, device=device, stream=stream, **kw)
    return fb.DeviceGraph.generate_rmat(fb.RmatParams(28, 16, seed=5), device=device, stream=stream, **kw)


def algorithmic_bytes(n: int, m: int) -> int:
    """Per iteration: 12 B/edge (int32 in_src + fp64 contrib
    gather) + 36 B/vertex (int64 row_ptr, pr read+write, int32 outdeg,
    contrib write)."""
    return 12 * m + 36 * n


def pb_stream_bytes(n: int, m: int, runs: int) -> int:
    """Per propagation-blocked sweep, what the two passes stream besides the
    random gather: 4 B source per edge; per run (one row's
    edges inside one source chunk, summed by the gather pass) 8 B partial sum
    written + 8 B read back + 2 B tile index + 2 B row key; + 36 B/vertex."""
    return 4 * m + 20 * runs + 36 * n


# Random 8-B fetches per second against the contribution vector's size,
# measured by bench_micro/gather_bench.cu (DESIGN.md §3 table).
GATHER_CEILING = ((33.6e6, 270e9), (134e6, 113e9), (537e6, 56e9), (2.15e9, 46e9))


def ceiling_ms(n: int, m: int, pb: bool, peak: float, runs: int = 0) -> float:
    """The sweep's own floor: the pull sweep's gathers at the measured random-
    fetch rate for 8 n bytes of contributions; a propagation-blocked sweep's
    gathers at ~270 G/s (one L2 request each, L2-resident window) plus the
    accumulate's stream (20 B/run + 36 B/vertex) at the copy peak."""
    if pb:
        return (m / 270e9 + (20 * runs + 36 * n) / (peak * 1e9)) * 1e3
    size = 8 * n
    rate = next((r for s, r in GATHER_CEILING if size <= s * 1.05), GATHER_CEILING[-1][1])
    return m / rate * 1e3


def ncu_traffic(key: str):
    """DRAM read+write bytes per unit from the committed ncu capture."""
    try:
        with open(os.path.join(ROOT, "profiles", "traffic.json")) as f:
            return json.load(f).get(key)
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


def host_threads() -> int:
    try:
        return len(os.sched_getaffinity(0))
    except Exception:
        return os.cpu_count() or 1


def cpu_model() -> str:
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except Exception:
        pass
    return "unknown"


# --------------------------------------------------------------- reference arm
def run_reference(args) -> None:
    """The unmodified reference (oracle/_ref) on the same workload: graph
    handed over from the device generator (bit-identical arrays), the
    reference's own build_layout in its graph handle (untimed), then ONE
    timed pagerank_ec_par call of REF_SAMPLE_ITERS iterations on every host
    thread (a full solve would take ~23 min on config 5)."""
    ws, rank, local = dist_env()
    if rank != 0:
        return
    from oracle import Graph as OGraph
    from oracle import load_reference

    ref = load_reference()
    threads = host_threads()
    config = args.workload
    if ref is None:
        print(json.dumps({"impl": "reference", "unavailable": "oracle/_ref/libfpr_ref.so not built"}), flush=True)
        return
    t0 = time.perf_counter()
    if config in ("1", "2"):  # small enough for the reference's own generators
        n0, s, d = ref.generate_rmat(16, 16, seed=1) if config == "1" else ref.random_sparse(1 << 22, 16, 2)
        og = ref.build_csr(n0, s, d)
        del s, d
    else:  # config 5: the device generator's arrays (the reference's would need ~175 GB and ~45 min)
        import paper_2203_09284_b200 as fb

        with make_graph(fb, config, local, pb=False) as dg:
            g = dg.download()
        og = OGraph(g.n, g.m, g.in_start, g.in_src, g.out_degree)
        del g
    h = ref.graph_handle(og)  # copies into fpr::Graph + the reference's build_layout
    n, m = og.n, og.m
    del og  # the reference holds its own copy
    setup_s = time.perf_counter() - t0
    iters = REF_SAMPLE_ITERS if config == "5" else 10000
    try:
        r = ref.run(OGraph(n, m, None, None, None), "ec_par", DAMPING, THRESHOLD, iters, threads, handle=h)
    finally:
        ref.destroy(h)
    gteps = m * r.iterations / r.seconds / 1e9
    sample = (f"one fpr::pagerank_ec_par call of {r.iterations} iterations on config 5, T={threads} "
              f"(a full solve is 54 iterations, ~23 min on 16 cores)" if config == "5" else
              f"one full fpr::pagerank_ec_par solve ({r.iterations} iterations), T={threads}")
    data = ("synthetic (device-generated arrays, bit-identical to generate_rmat+build_csr)" if config == "5"
            else "synthetic (the reference's own generator + build_csr)")
    line = {"metric": METRIC, "value": gteps, "unit": "GTEPS", "impl": "reference", "n_gpus": ws,
            "steps": 1, "warmup": 0, "requested_steps": args.steps, "requested_warmup": args.warmup,
            "ms_per_step": 1e3 * r.seconds, "higher_is_better": True, "scaling": "strong", "vs_baseline": None,
            "dtype": "f64", "data": data, "config": config_block(config, n, m),
            "step": (f"bounded sample: {r.iterations} EC iterations in one pagerank_ec_par call (GTEPS/iter)"
                     if config == "5" else "1 full EC solve (time-to-converge)"), "iterations_timed": r.iterations,
            "cpu_baseline": {"value": gteps, "unit": "GTEPS", "cores": threads, "kind": "reference",
                             "cpu": cpu_model(), "sample": sample, "setup_s_untimed": setup_s},
            "e2e": {"value": gteps, "unit": "GTEPS", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


def config_block(config: str, n: int, m: int) -> dict:
    return {"workload": WORKLOADS[config], "n": n, "m": m, "threshold": THRESHOLD, "norm": "linf",
            "damping": DAMPING,
            "l2": {"5": "inputs larger than L2 (in_src 17 GB, contributions 2.1 GB); no flush",
                   "2": "in_src 268 MB > L2; contributions L2-resident; no flush",
                   "1": "L2-resident (correctness-sized config)"}[config]}


# ----------------------------------------------------------- CPU baselines
def reference_engines(ref, og, threads, full=True, sample_iters=2, reps=2) -> dict:
    """The reference's four engines (pagerank.hpp:128,156,195,261) on one
    graph handle (build_layout excluded): time-to-converge as
    the min over `reps` when `full`, else s/iter over a bounded
    sample of `sample_iters` iterations."""
    out = {}
    h = ref.graph_handle(og)
    try:
        for eng in ("ec_seq", "fused_seq", "ec_par", "fused_par"):
            t = threads if eng.endswith("par") else 1
            if full:
                runs = [ref.run(og, eng, DAMPING, THRESHOLD, 10000, t, handle=h)
                        for _ in range(reps if eng.endswith("par") else 1)]
                best = min(runs, key=lambda x: x.seconds)
                out[eng] = {"time_to_converge_s": best.seconds, "iterations": best.iterations, "threads": t,
                            "reps": len(runs), "gteps": og.m * best.iterations / best.seconds / 1e9,
                            "iterations_all_reps": [x.iterations for x in runs]}
            else:
                r = ref.run(og, eng, DAMPING, THRESHOLD, sample_iters, t, handle=h)
                out[eng] = {"s_per_iter": r.seconds / r.iterations, "iterations_timed": r.iterations,
                            "threads": t, "gteps": og.m * r.iterations / r.seconds / 1e9}
    finally:
        ref.destroy(h)
    return out


def cpu_baseline_leg(fb, device, g5, gpu_iter1) -> dict:
    """Rank 0, N=1, on the GPU box's host cores.
      * value: the oracle port's EC iteration on config 5 (fo_ec_step, the
        reference's iteration in pull form, OpenMP over every host thread;
        ~10-20 s), its result also a live parity check of the GPU's first
        iterate;
      * reference_engines: the unmodified reference (oracle/_ref) on config 2
        (all four engines, full solves, min over repetitions) and config 3
        (bounded: 2 iterations each; the full runs' iteration counts are in
        tests/golden/config3.json);
      * the reference on config 5 itself is the --impl reference arm."""
    from oracle import Graph as OGraph
    from oracle import Oracle, load_reference

    threads = host_threads()
    o = Oracle()
    og5 = OGraph(g5.n, g5.m, g5.in_start, g5.in_src, g5.out_degree)
    t0 = time.perf_counter()
    nxt, err, _ = o.ec_step(og5, np.full(g5.n, 1.0 / g5.n), DAMPING)
    dt = time.perf_counter() - t0
    out = {"value": g5.m / dt / 1e9, "unit": "GTEPS", "cores": threads, "kind": "port", "cpu": cpu_model(),
           "sample": "1 EC iteration of config 5 with the oracle port (fo_ec_step: scatter+gather of "
                     "pagerank.hpp:137-140 in pull form, OpenMP over rows)",
           "seconds": dt}
    if gpu_iter1 is not None:
        out["parity_iter1_max_rel"] = float(np.max(np.abs(gpu_iter1 - nxt) / nxt))
    del nxt
    ref = load_reference()
    if ref is None:
        out["reference_engines"] = {"unavailable": "oracle/_ref not built"}
        return out
    eng = {}
    for config, full in (("2", True), ("3", False)):
        with make_graph(fb, config, device, pb=False) as dg:
            g = dg.download()
        og = OGraph(g.n, g.m, g.in_start, g.in_src, g.out_degree)
        eng["config" + config] = {"n": g.n, "m": g.m, "mode": "full solves" if full else "2-iteration samples",
                                  **reference_engines(ref, og, threads, full=full)}
        del g, og
    eng["engine"] = "oracle/_ref: the unmodified reference headers, -O3 (reference Release flags), T = host threads"
    out["reference_engines"] = eng
    return out


# ------------------------------------------------------------ secondary legs
def secondary_legs(fb, device, peak) -> dict:
    """Configs 2-4 (and config 5's FusEd), generated on the device (untimed):
    EC and FusEd time-to-converge (CUDA-event solve times), ms per sweep,
    GTEPS and the BASELINE roofline fraction, each on the sweep the library
    picks by default.  Not the headline; reported beside it."""
    cfg = fb.PageRankConfig(damping=DAMPING, threshold=THRESHOLD)
    out = {}

    def record(dg, r):
        ms_it = r.solve_ms / r.trace.iterations
        pb = r.sweep == fb.SWEEP_PB
        return {"iterations": r.trace.iterations, "converged": bool(r.trace.converged),
                "time_to_converge_ms": r.solve_ms, "ms_per_sweep": ms_it, "gteps": dg.m / ms_it / 1e6,
                "roofline_frac": algorithmic_bytes(dg.n, dg.m) / (ms_it * 1e-3) / 1e9 / peak,
                "sweep": "pb" if pb else "pull",
                # the sweep's own ceiling: pull = the measured random-fetch
                # rate for a contribution vector of this size; PB = gather requests + stream
                "ceiling_ms": ceiling_ms(dg.n, dg.m, pb, peak, dg.layout_info()["runs"]),
                "ceiling_frac": ceiling_ms(dg.n, dg.m, pb, peak, dg.layout_info()["runs"]) / ms_it}

    names = {"2": "config2: uniform G(n=2^22, 2^26 draws, seed 2)",
             "3": "config3: RMAT s24 ef16 seed 3, BFS crawl-order relabel",
             "4": "config4: Chung-Lu n=2^26, 1.2e9 draws, alpha 2.1, seed 4, random order"}
    for c in ("2", "3", "4"):
        with make_graph(fb, c, device) as dg:
            rec = {"workload": names[c], "n": dg.n, "m": dg.m}
            for eng, tag in ((fb.ENGINE_EC, "ec"), (fb.ENGINE_FUSED, "fused"),
                             (fb.ENGINE_FUSED_LOCKSTEP, "lockstep")):
                dg.run(eng, cfg, copy_ranks=False, copy_trace=False)  # one-time layouts / wave plans
                rec[tag] = record(dg, dg.run(eng, cfg, copy_ranks=False, copy_trace=False))
            if c == "2":
                # BASELINE words the stop rule as an L1 delta; same graph, L1 rule
                with make_graph(fb, c, device, norm=fb.NORM_L1) as d1:
                    r1 = d1.run(fb.ENGINE_EC, cfg, copy_ranks=False, copy_trace=False)
                    rec["ec_l1_stop_rule"] = {"iterations": r1.trace.iterations, "time_to_converge_ms": r1.solve_ms}
            out["config" + c] = rec
    return out


# ------------------------------------------------------------------ main arm
def main() -> None:
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--workload", default="5", choices=sorted(WORKLOADS), help="headline graph (default config 5)")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-large", action="store_true", help="skip the secondary configs 2-4 legs")
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
    if ws > 1 or args.partitioned:
        import torch.distributed as dist

        if ws == 1:
            os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
            os.environ.setdefault("MASTER_PORT", "29531")
            os.environ.setdefault("RANK", "0")
            os.environ.setdefault("WORLD_SIZE", "1")
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        run_multi(args, fb, dist, ws, rank, local)
        dist.destroy_process_group()
        return
    stream = torch.cuda.current_stream()
    sptr = fb.torch_stream_handle()
    peak, peak_kind = peaks()

    dg = make_graph(fb, args.workload, local, stream=sptr)
    n, m = dg.n, dg.m
    cfg = fb.PageRankConfig(damping=DAMPING, threshold=THRESHOLD)

    def step():
        return dg.run(fb.ENGINE_EC, cfg, copy_ranks=False, copy_trace=False)

    t_first = time.perf_counter()
    first = step()  # builds the sweep's one-time layout (propagation blocking on config 5)
    torch.cuda.synchronize()
    first_s = time.perf_counter() - t_first
    for _ in range(args.warmup - 1):
        r = step()
    iters = first.trace.iterations
    launches_per_step = first.kernel_launches

    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    kernel_ms = []
    with ClockSampler(local) as clk:
        torch.cuda.synchronize()
        ev0.record(stream)
        for _ in range(args.steps):
            r = step()
            kernel_ms.append(r.solve_ms)
            assert r.trace.iterations == iters
        ev1.record(stream)
        torch.cuda.synchronize()
    ms_step = ev0.elapsed_time(ev1) / args.steps
    value = m * iters / (ms_step * 1e-3) / 1e9
    kms = float(np.mean(kernel_ms))  # CUDA-event time of the sweeps (the library's stream = torch's)
    sweep_ms = kms / iters
    achieved = algorithmic_bytes(n, m) / (sweep_ms * 1e-3) / 1e9
    pb = r.sweep == fb.SWEEP_PB
    runs = dg.layout_info()["runs"]

    # per-iteration device times and trace of one more solve
    tr = dg.run(fb.ENGINE_EC, cfg, copy_ranks=True, copy_trace=True)
    it_ms = (tr.trace.iter_ns.astype(np.float64) / 1e6).tolist()
    # FusEd on the same resident graph (the library's FUSED choice: the
    # lockstep Gauss-Seidel schedule on PB sweeps here)
    fr = dg.run(fb.ENGINE_FUSED, cfg, copy_ranks=False, copy_trace=False)
    fr = dg.run(fb.ENGINE_FUSED, cfg, copy_ranks=False, copy_trace=False)
    fused = {"iterations": fr.trace.iterations, "time_to_converge_ms": fr.solve_ms,
             "ms_per_sweep": fr.solve_ms / fr.trace.iterations, "sweep": "pb" if fr.sweep == fb.SWEEP_PB else "pull",
             "schedule": "wave-lockstep Gauss-Seidel" if fr.sweep == fb.SWEEP_PB else "block-asynchronous",
             "waves": int(len(dg.wave_starts()) - 1)}
    # the pull sweep on the same graph, for comparison (forced)
    pull = None
    if not args.no_large and args.workload == "5":
        with make_graph(fb, args.workload, local, stream=sptr, pb=False) as dp:
            rp = dp.run(fb.ENGINE_EC, cfg, copy_ranks=False, copy_trace=False)
            pull = {"iterations": rp.trace.iterations, "time_to_converge_ms": rp.solve_ms,
                    "ms_per_sweep": rp.solve_ms / rp.trace.iterations,
                    "roofline_frac": algorithmic_bytes(n, m) / (rp.solve_ms / rp.trace.iterations * 1e-3) / 1e9 / peak}
    # the opt-in renumbering by degree inside each source chunk
    # (FPR_B200_OPT_REORDER_BLOCKS): faster sweeps, paid by a CSR rebuild at creation
    reorder = None
    if not args.no_large and args.workload == "5":
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        with make_graph(fb, args.workload, local, stream=sptr, reorder="blocks") as dr:
            torch.cuda.synchronize()
            create_s = time.perf_counter() - t0
            dr.run(fb.ENGINE_EC, cfg, copy_ranks=False, copy_trace=False)  # the layout
            re_ec = dr.run(fb.ENGINE_EC, cfg, copy_ranks=False, copy_trace=False)
            re_fu = dr.run(fb.ENGINE_FUSED, cfg, copy_ranks=False, copy_trace=False)
        reorder = {"option": "FPR_B200_OPT_REORDER_BLOCKS", "iterations": re_ec.trace.iterations,
                   "time_to_converge_ms": re_ec.solve_ms, "ms_per_sweep": re_ec.solve_ms / re_ec.trace.iterations,
                   "gteps": m * re_ec.trace.iterations / re_ec.solve_ms / 1e6,
                   "fused_iterations": re_fu.trace.iterations, "fused_time_to_converge_ms": re_fu.solve_ms,
                   "create_s_with_generation": create_s}

    g_host = None
    e2e = None
    keep = None
    if not args.no_e2e or not args.no_cpu_baseline:
        keep = pinned_csr(torch, n, m)
        dg.download_into(*(k[1] for k in keep))
        g_host = fb.Graph(n, m, keep[0][1], keep[1][1], keep[2][1])
    gpu_iter1 = None
    if not args.no_cpu_baseline:
        gpu_iter1 = dg.run(fb.ENGINE_EC, fb.PageRankConfig(damping=DAMPING, threshold=THRESHOLD, max_iterations=1),
                           copy_ranks=True, copy_trace=False).ranks.values
    dg.close()
    if not args.no_e2e:
        e2e = e2e_leg(fb, g_host, local, args, iters)
    large = None if args.no_large else secondary_legs(fb, local, peak)
    cpu = None
    if not args.no_cpu_baseline:
        cpu = cpu_baseline_leg(fb, local, g_host, gpu_iter1)

    traffic = ncu_traffic("config5_ec_pb_sweep" if pb else "config5_ec_pull_sweep")
    line = {
        "metric": METRIC, "value": value, "unit": "GTEPS",
        "n_gpus": ws, "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms_step,
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (device-generated, bit-identical to reference generate_rmat+build_csr)",
        "config": config_block(args.workload, n, m),  # the reference arm prints the same block
        "step": "1 full EC solve (time-to-converge)", "iterations": iters, "parallelism": "single-gpu",
        "sweep": "propagation-blocked (the library's default for this graph)" if pb else "pull (library default)",
        "time_to_converge_ms": ms_step,
        "first_solve_s_with_layout_build": first_s,
        "iteration_ms": it_ms,
        "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s", "frac": achieved / peak,
                     "traffic": traffic.get("dram_bytes_per_sweep") if traffic else None, "peak_kind": peak_kind,
                     "unit_of_work": "one EC sweep (the PB gather + accumulate + reduce launches) = one iteration",
                     "algorithmic_bytes_per_sweep": algorithmic_bytes(n, m),
                     "sweep_ms": sweep_ms,
                     "pb_runs": runs if pb else None,
                     "pb_stream_bytes_frac": (pb_stream_bytes(n, m, runs) / (sweep_ms * 1e-3) / 1e9 / peak
                                              if pb else None),
                     # the design's own floor: the gather pass at the measured
                     # random-fetch ceiling (~270 G L2 requests/s, bench_micro/gather_bench.cu)
                     # plus the accumulate's stream (20 B/run + 36 B/vertex) at the copy peak
                     "pb_design_floor_ms": ceiling_ms(n, m, True, peak, runs) if pb else None,
                     "pb_design_floor_frac": ceiling_ms(n, m, True, peak, runs) / sweep_ms if pb else None,
                     "traffic_source": traffic.get("source") if traffic else None,
                     "kernel_shares": traffic.get("kernel_shares") if traffic else None},
        "fused": fused,
        "ec_pull_sweep": pull,
        "ec_reorder_blocks": reorder,
        "cpu_baseline": cpu,
        "e2e": e2e,
        "configs_2_4": large,
        "gpu_launches": int(launches_per_step * args.steps),
        "clocks": clk.summary(),
    }
    print(json.dumps(line), flush=True)


def pinned_csr(torch, n, m):
    def pinned(k):
        t = torch.empty(k, dtype=torch.int64, pin_memory=True)
        return t, t.numpy().view(np.uint64)

    return [pinned(n + 1), pinned(max(m, 1)), pinned(n)]


def e2e_leg(fb, g, device, args, iters) -> dict:
    """fpr_b200_pagerank() on pinned host fpr::Graph arrays (u64); H2D +
    narrowing + partition + the one-time sweep layout + solve + D2H of ranks
    and error trace, all inside the timed call."""
    import torch

    ranks_t = torch.empty(g.n, dtype=torch.float64, pin_memory=True)
    errs_t = torch.empty(10000, dtype=torch.float64, pin_memory=True)
    view = fb._GraphView(g.n, g.m, g.in_start.ctypes.data, g.in_src.ctypes.data, g.out_degree.ctypes.data)
    cfg = fb.PageRankConfig(damping=DAMPING, threshold=THRESHOLD)._c()
    opts = fb._options(device=device, stream=fb.torch_stream_handle())
    res = fb._Result()
    L = fb.lib()

    def call():
        fb._check(L.fpr_b200_pagerank(C.byref(view), fb.ENGINE_EC, C.byref(cfg), C.byref(opts),
                                      ranks_t.data_ptr(), errs_t.data_ptr(), 10000, C.byref(res)))

    call()
    steps = max(2, min(args.steps, 3))
    torch.cuda.synchronize()
    times = []
    for _ in range(steps):
        t0 = time.perf_counter()
        call()
        torch.cuda.synchronize()
        times.append(time.perf_counter() - t0)
    dt = float(np.mean(times))
    assert res.iterations == iters
    h2d = 8 * (g.n + 1) + 8 * g.m + 8 * g.n
    d2h = 8 * g.n + 8 * int(res.iterations)
    return {"value": g.m * res.iterations / dt / 1e9, "unit": "GTEPS", "h2d_bytes_per_step": h2d,
            "d2h_bytes_per_step": d2h, "ms_per_step": dt * 1e3, "steps": steps,
            "sweep": "pb" if res.sweep == fb.SWEEP_PB else "pull",
            "api": "fpr_b200_pagerank (C ABI, pinned host u64 CSR; sweep layout built inside every call)"}


# ------------------------------------------------------------------ N GPUs
def run_multi(args, fb, dist, ws, rank, local) -> None:
    """N GPUs: destination-range partition of the headline graph (strong
    scaling), one residual all-gather per iteration, contributions exchanged
    by the sweep's own P2P stores (paper_2203_09284_b200/dist.py)."""
    import torch

    from paper_2203_09284_b200.dist import B200Part, PartitionedSolver, TorchExchange

    sptr = fb.torch_stream_handle()
    full = make_graph(fb, args.workload, local, stream=sptr, pb=False)
    n, m = full.n, full.m
    part = B200Part(full, ws, rank, device=local, stream=sptr)
    full.close()
    ex = TorchExchange()
    cfg = fb.PageRankConfig(damping=DAMPING, threshold=THRESHOLD)
    dev = f"cuda:{local}"
    solver = PartitionedSolver(part, ex, device=dev, fused_exchange=not args.copy_exchange and ws > 1,
                               device_stop=True, batch=8)
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
    exchange = ("fused: sweep epilogue P2P-stores each slice into the peers' replicas (CUDA IPC over NVLink); "
                "NCCL all-gather of the 16-B residual pair" if solver.fused_exchange else
                "NCCL all-gather of contribution slices + residual pair")
    peak, _ = peaks()
    sweep_ms = ms_step / iters
    if rank == 0:
        line = {
            "metric": METRIC, "value": m * iters / (ms_step * 1e-3) / 1e9, "unit": "GTEPS", "n_gpus": ws,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms_step,
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic (device-generated, bit-identical to reference generate_rmat+build_csr)",
            "config": config_block(args.workload, n, m),
            "step": "1 full EC solve (time-to-converge)",
            "iterations": iters, "parallelism": f"dst-range partition x{ws}", "exchange": exchange,
            "sweep": ("propagation-blocked" if part.graph.layout_info()["sweep"] == fb.SWEEP_PB else "pull")
                     + " (per part, the library's choice for the part's exchange space)",
            "host_loop": ("device-side stop: batches of 8 iterations (sweep, pair all-gather, gate update) "
                          "enqueued without a host read; one gate read per batch"),
            "exchange_fallback": solver.fallback, "slice": part.slice,
            "time_to_converge_ms": ms_step,
            "fused": {"iterations": fr.iterations},
            "roofline": {"bound": "hbm", "achieved": algorithmic_bytes(n, m) / ws / (sweep_ms * 1e-3) / 1e9,
                         "peak": peak, "unit": "GB/s (per GPU)",
                         "frac": algorithmic_bytes(n, m) / ws / (sweep_ms * 1e-3) / 1e9 / peak, "traffic": None},
            "cpu_baseline": None, "e2e": None,
            # per issued sweep (batches of 8, the ones past the stop are no-ops): the PB
            # sweep's hot-copy refresh, gather, accumulate and reduce (or the pull
            # solve kernel) + the gate update
            "gpu_launches": int(args.steps * ((iters + 7) // 8 * 8) *
                                ((5 if part.graph.layout_info()["sweep"] == fb.SWEEP_PB else 2))),
            "clocks": clk.summary(),
        }
        print(json.dumps(line), flush=True)
    solver.close()
    part.close()


if __name__ == "__main__":
    main()
