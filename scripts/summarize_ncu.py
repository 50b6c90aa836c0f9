"""Summarise ncu artefacts for profiles/: python scripts/summarize_ncu.py <launches.csv> <full.ncu-rep> <out.md> [algorithmic_bytes_per_launch]"""
import csv, io, subprocess, sys
from collections import defaultdict

launches, rep, out = sys.argv[1:4]
alg = float(sys.argv[4]) if len(sys.argv) > 4 else None
lines = []
rows = [r for r in csv.reader(open(launches)) if len(r) > 5]
h = rows[0]
iN, iV, iU = h.index("Kernel Name"), h.index("Metric Value"), h.index("Metric Unit")
agg = defaultdict(lambda: [0, 0.0])
for r in rows[1:]:
    v = float(r[iV].replace(",", ""))
    v = v / 1e3 if r[iU] == "ns" else (v * 1e3 if r[iU] == "ms" else v)
    agg[r[iN].split("(")[0][:70]][0] += 1
    agg[r[iN].split("(")[0][:70]][1] += v
tot = sum(x[1] for x in agg.values())
lines.append("## Launch list (ncu gpu__time_duration.sum, --clock-control none; cold-cache, serialised)\n")
lines.append("| launches | total us | share | kernel |\n|---:|---:|---:|---|")
for k, (c, t) in sorted(agg.items(), key=lambda x: -x[1][1]):
    lines.append(f"| {c} | {t:.1f} | {100 * t / tot:.1f}% | `{k}` |")
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
r = list(csv.reader(io.StringIO(raw)))
hh, uu, vv = r[0], r[1], r[2]
d = {hh[i]: (vv[i], uu[i]) for i in range(len(hh))}
want = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "dram__throughput.avg.pct_of_peak_sustained_elapsed", "lts__t_sector_hit_rate.pct",
        "lts__t_sectors_srcunit_tex_op_read.sum", "lts__throughput.avg.pct_of_peak_sustained_elapsed",
        "l1tex__throughput.avg.pct_of_peak_sustained_elapsed",
        "l1tex__m_l1tex2xbar_req_cycles_active.avg.pct_of_peak_sustained_elapsed",
        "l1tex__t_output_wavefronts_pipe_lsu_mem_global_op_ld.sum", "smsp__inst_executed.sum",
        "smsp__issue_active.avg.pct_of_peak_sustained_active", "sm__warps_active.avg.pct_of_peak_sustained_active",
        "launch__registers_per_thread", "launch__grid_size", "launch__block_size"]
lines.append("\n## Full capture of the top kernel (ncu --set full, one launch)\n")
lines.append(f"Kernel: `{r[2][hh.index('Kernel Name')] if 'Kernel Name' in hh else '?'}`\n")
lines.append("| metric | value | unit |\n|---|---:|---|")
for k in want:
    if k in d:
        lines.append(f"| {k} | {d[k][0]} | {d[k][1]} |")
def num(k):
    x, u = d[k]
    x = float(x.replace(",", ""))
    return x * {"Gbyte": 1e9, "Mbyte": 1e6, "Kbyte": 1e3, "byte": 1}.get(u, 1)
traffic = num("dram__bytes_read.sum") + num("dram__bytes_write.sum")
lines.append(f"\nDRAM traffic per launch (read+write): {traffic / 1e9:.3f} GB")
if alg:
    lines.append(f"Algorithmic bytes per launch: {alg / 1e9:.3f} GB (traffic/algorithmic = {traffic / alg:.2f})")
stalls = sorted(((float(d[k][0].replace(",", "") or 0), k) for k in hh
                 if "pcsamp_warps_issue_stalled" in k and not k.endswith("not_issued")), reverse=True)
tots = sum(s for s, _ in stalls) or 1
lines.append("\n## Warp stall sampling (top)\n")
for s, k in stalls[:8]:
    lines.append(f"- {k.replace('smsp__pcsamp_warps_issue_stalled_', '')}: {100 * s / tots:.1f}%")
open(out, "w").write("\n".join(lines) + "\n")
print("\n".join(lines))
