"""Summarise ncu captures into profiles/<round>/ text files (run in the build container).

    python tools/summarize_profiles.py r01 gpurun_out/prof_query.ncu-rep ...
    python tools/summarize_profiles.py r01 --launches gpurun_out/launches.csv
"""

import csv
import io
import os
import subprocess
import sys
from collections import defaultdict

METRICS = [
    ("gpu__time_duration.sum", "duration"),
    ("sm__cycles_elapsed.avg.per_second", "sm clock (Hz)"),
    ("dram__bytes_read.sum", "dram read bytes"),
    ("dram__bytes_write.sum", "dram write bytes"),
    ("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "dram throughput % of peak"),
    ("dram__throughput.avg.pct_of_peak_sustained_elapsed", "dram throughput %"),
    ("sm__throughput.avg.pct_of_peak_sustained_elapsed", "SM throughput %"),
    ("sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active", "tensor pipe active %"),
    ("sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active", "XU (MUFU) pipe %"),
    ("sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active", "FMA pipe %"),
    ("sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active", "ALU pipe %"),
    ("sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active", "FP64 pipe %"),
    ("sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active", "LSU pipe %"),
    ("sm__issue_active.avg.pct_of_peak_sustained_active", "issue active %"),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "achieved occupancy %"),
    ("launch__registers_per_thread", "registers / thread"),
    ("launch__shared_mem_per_block_dynamic", "dynamic smem / block"),
    ("launch__grid_size", "grid"),
    ("launch__block_size", "block"),
    ("smsp__inst_executed.sum", "warp instructions"),
]


def raw_metrics(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                         text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units, vals = rows[0], rows[1], rows[2]
    return {h: (v, u) for h, u, v in zip(hdr, units, vals)}


def stall_summary(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                         text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, vals = rows[0], rows[2]
    st = {}
    for h, v in zip(hdr, vals):
        if h.startswith("smsp__pcsamp_warps_issue_stalled_") and not h.endswith("not_issued"):
            try:
                st[h.replace("smsp__pcsamp_warps_issue_stalled_", "")] = float(v)
            except ValueError:
                pass
    tot = sum(st.values()) or 1.0
    return sorted(((k, v / tot) for k, v in st.items()), key=lambda kv: -kv[1])[:8]


def summarize(rep, round_dir):
    m = raw_metrics(rep)
    name = subprocess.run(["ncu", "-i", rep, "--page", "details", "--csv"], capture_output=True,
                          text=True).stdout.splitlines()
    kname = ""
    for line in name[1:2]:
        kname = next(csv.reader([line]))[4] if line else ""
    lines = [f"# ncu --set full summary: {os.path.basename(rep)}", f"kernel: {kname}", ""]
    for key, label in METRICS:
        if key in m:
            v, u = m[key]
            lines.append(f"{label:32s} {v} {u}")
    rd = m.get("dram__bytes_read.sum", ("0", ""))
    wr = m.get("dram__bytes_write.sum", ("0", ""))
    try:
        scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
        tr = float(rd[0].replace(",", "")) * scale.get(rd[1], 1) + \
            float(wr[0].replace(",", "")) * scale.get(wr[1], 1)
        lines.append(f"{'dram traffic (read+write)':32s} {tr:.4g} bytes")
    except (ValueError, KeyError):
        pass
    lines.append("")
    lines.append("top warp stall reasons (share of PC samples):")
    for k, f in stall_summary(rep):
        lines.append(f"  {k:28s} {100 * f:5.1f}%")
    out = os.path.join(round_dir, os.path.basename(rep).replace(".ncu-rep", ".txt"))
    with open(out, "w") as fh:
        fh.write("\n".join(lines) + "\n")
    print(out)


def launches(csv_path, round_dir):
    rows = list(csv.reader(open(csv_path)))
    start = next(i for i, r in enumerate(rows) if r and r[0] == "ID")
    hdr = rows[start]
    ki, vi, ui = hdr.index("Kernel Name"), hdr.index("Metric Value"), hdr.index("Metric Unit")
    agg = defaultdict(list)
    unit = ""
    for r in rows[start + 1:]:
        if len(r) > vi:
            agg[r[ki]].append(float(r[vi].replace(",", "")))
            unit = r[ui]
    total = sum(sum(v) for v in agg.values())
    lines = ["# launch list (ncu --metrics gpu__time_duration.sum --clock-control none)",
             "# cold-cache, serialised: compare shares, not absolutes", "",
             f"{'launches':>8s} {'mean':>12s} {'share':>7s}  kernel"]
    for k, v in sorted(agg.items(), key=lambda kv: -sum(kv[1])):
        lines.append(f"{len(v):8d} {sum(v) / len(v):10.1f}{unit:>2s} {100 * sum(v) / total:6.1f}%  {k[:110]}")
    out = os.path.join(round_dir, "launches_summary.txt")
    with open(out, "w") as fh:
        fh.write("\n".join(lines) + "\n")
    print(out)


if __name__ == "__main__":
    rnd = sys.argv[1]
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    rdir = os.path.join(root, "profiles", rnd)
    os.makedirs(rdir, exist_ok=True)
    args = sys.argv[2:]
    if args and args[0] == "--launches":
        launches(args[1], rdir)
    else:
        for rep in args:
            summarize(rep, rdir)
