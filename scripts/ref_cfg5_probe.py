"""Box probe: can the unmodified reference (oracle/_ref) run config 5 here?
Prints host RAM / cores, then (if RAM allows) times graph hand-off,
build_layout and a few ec_par iterations on the device-generated config 5."""
import json
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def meminfo():
    d = {}
    for line in open("/proc/meminfo"):
        k, v = line.split(":")
        d[k] = int(v.split()[0]) * 1024
    return d


def rss():
    for line in open("/proc/self/status"):
        if line.startswith("VmRSS") or line.startswith("VmHWM"):
            print(line.strip(), flush=True)


mi = meminfo()
print(json.dumps({"mem_total_gb": mi["MemTotal"] / 1e9, "mem_avail_gb": mi["MemAvailable"] / 1e9,
                  "nproc": os.cpu_count(), "affinity": len(os.sched_getaffinity(0))}), flush=True)
scale = int(sys.argv[1]) if len(sys.argv) > 1 else 28
need = (16 << scale) * 8 * 5  # u64 in_src python + copy + layout(2x) + slack
if mi["MemAvailable"] < need:
    print(f"not enough host RAM for scale {scale}: need ~{need / 1e9:.0f} GB", flush=True)
    sys.exit(0)
import paper_2203_09284_b200 as fb
from oracle import load_reference

ref = load_reference()
t0 = time.time()
dg = fb.DeviceGraph.generate_rmat(fb.RmatParams(scale, 16, seed=5), device=0)
print("gen", time.time() - t0, dg.n, dg.m, flush=True)
t0 = time.time()
g = dg.download()
dg.close()
print("download", time.time() - t0, flush=True)
rss()
t0 = time.time()
h = ref.graph_handle(g)
print("ref_graph_create (copy + build_layout)", time.time() - t0, flush=True)
rss()
threads = len(os.sched_getaffinity(0))
for k in (1, 2, 3):
    r = ref.run(g, "ec_par", 0.85, 1e-10, k, threads, handle=h)
    print(f"ec_par max_iter={k} threads={threads}: {r.seconds:.3f} s", flush=True)
r = ref.run(g, "fused_par", 0.85, 1e-10, 2, threads, handle=h)
print(f"fused_par max_iter=2: {r.seconds:.3f} s", flush=True)
r = ref.run(g, "ec_seq", 0.85, 1e-10, 1, 1, handle=h)
print(f"ec_seq max_iter=1: {r.seconds:.3f} s", flush=True)
rss()
