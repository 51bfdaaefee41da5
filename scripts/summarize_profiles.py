"""Summaries of ncu captures for profiles/ (run here, on the CPU box).

  python scripts/summarize_profiles.py TAG OUTPREFIX
reads gpurun_out/TAG_{p2p,m2l}_raw.csv, TAG_launches.csv, TAG_pipe_launches.csv
and writes OUTPREFIX_ncu_summary.json + OUTPREFIX_launches.txt.
"""
import csv
import json
import sys
from collections import defaultdict

tag, out = sys.argv[1], sys.argv[2]
G = "gpurun_out/"
WANT = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active",
        "sm__throughput.avg.pct_of_peak_sustained_elapsed",
        "smsp__issue_active.avg.pct_of_peak_sustained_active",
        "sm__warps_active.avg.pct_of_peak_sustained_active",
        "launch__registers_per_thread", "launch__occupancy_limit_registers",
        "lts__t_sector_hit_rate.pct", "smsp__inst_executed.sum",
        "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active",
        "l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_ld.sum",
        "launch__grid_size", "launch__block_size"]
STALLS = ["math_pipe_throttle", "wait", "not_selected", "selected", "long_scoreboard",
          "short_scoreboard", "dispatch_stall", "branch_resolving", "no_instruction",
          "mio_throttle", "barrier", "membar", "lg_throttle"]


def raw(kind):
    rows = list(csv.reader(open(f"{G}{tag}_{kind}_raw.csv")))
    h, u, v = rows[0], rows[1], rows[2]
    d = {"kernel": v[h.index("Kernel Name")]}
    for w in WANT:
        if w in h:
            d[w] = f"{v[h.index(w)]} {u[h.index(w)]}".strip()
    st = {}
    for s in STALLS:
        k = f"smsp__average_warps_issue_stalled_{s}_per_issue_active.ratio"
        if k in h:
            st[s] = float(v[h.index(k)])
    d["stall_cycles_per_issue"] = st
    return d


def launches(fname, keep_last_frac=1.0):
    rows = list(csv.reader(open(G + fname)))
    hdr = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
    h = rows[hdr]
    ki, vi = h.index("Kernel Name"), h.index("Metric Value")
    data = rows[hdr + 1:]
    data = data[int(len(data) * (1 - keep_last_frac)):]
    agg = defaultdict(lambda: [0, 0.0])
    for r in data:
        name = r[ki].split("(")[0].replace("void ", "")
        agg[name][0] += 1
        agg[name][1] += float(r[vi].replace(",", "")) / 1e6
    tot = sum(v[1] for v in agg.values())
    lines = [f"{'ms':>9} {'share':>6} {'n':>5}  kernel", "-" * 80]
    for k, (n, ms) in sorted(agg.items(), key=lambda x: -x[1][1]):
        lines.append(f"{ms:9.3f} {100 * ms / tot:5.1f}% {n:5d}  {k}")
    lines.append(f"{tot:9.3f}  total")
    return "\n".join(lines)


summary = {"tag": tag, "p2p_kernel": raw("p2p"), "m2l_thread_kernel": raw("m2l")}
json.dump(summary, open(f"{out}_ncu_summary.json", "w"), indent=1)
with open(f"{out}_launches.txt", "w") as f:
    f.write(f"# ncu --metrics gpu__time_duration.sum --clock-control none (cold-cache, serialised)\n")
    f.write(f"# (1) python bench.py --no-e2e --no-fmm --no-cpu --steps 3 --warmup 3  (config 4, 10M, L=10)\n")
    f.write(launches(f"{tag}_launches.csv") + "\n\n")
    f.write("# (2) one device-pipeline FmmEngine evaluate at 10M (second of two reps)\n")
    f.write(launches(f"{tag}_pipe_launches.csv", 0.5) + "\n")
print(open(f"{out}_launches.txt").read())
print(json.dumps(summary, indent=1))
