#!/usr/bin/env python
"""Summarise an ncu report (--set full) or a launch list (--metrics
gpu__time_duration.sum) into the text committed under profiles/.

  python tools/ncu_summary.py report.ncu-rep > profiles/<name>.txt
  python tools/ncu_summary.py --launches launches.csv > profiles/<name>.txt
"""
import csv
import io
import subprocess
import sys
from collections import defaultdict

KEYS = [
    "gpu__time_duration.sum", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
    "dram__bytes_read.sum", "dram__bytes_write.sum",
    "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
    "sm__pipe_tensor_subpipe_imma_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_tensor_subpipe_imma.avg.pct_of_peak_sustained_active",
    "TPC.TriageCompute.sm__pipe_tensor_cycles_active_realtime.avg.pct_of_peak_sustained_elapsed",
    "SM_A.TriageCompute.sm__inst_executed_pipe_xu_realtime.avg.pct_of_peak_sustained_elapsed",
    "sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_fmaheavy.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active",
    "smsp__issue_active.avg.pct_of_peak_sustained_active",
    "smsp__inst_issued.sum", "sm__warps_active.avg.pct_of_peak_sustained_active",
    "launch__registers_per_thread", "launch__grid_size", "launch__block_size",
    "smsp__average_warp_latency_per_inst_issued.ratio",
]


def report(path):
    raw = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True,
                         text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    hdr, units = rows[0], rows[1]
    for vals in rows[2:]:
        d = dict(zip(hdr, vals))
        print(f"kernel: {d.get('Kernel Name', '?')[:100]}")
        for k in KEYS:
            if k in d:
                print(f"  {k:95s} {d[k]:>16s} {units[hdr.index(k)]}")
        stalls = []
        for h, v in zip(hdr, vals):
            if h.startswith("smsp__pcsamp_warps_issue_stalled_") and not h.endswith("_not_issued"):
                try:
                    stalls.append((float(v.replace(",", "")), h))
                except ValueError:
                    pass
        tot = sum(s for s, _ in stalls) or 1.0
        print("  top stall reasons (pc sampling):")
        for s, h in sorted(stalls, reverse=True)[:8]:
            print(f"    {h.replace('smsp__pcsamp_warps_issue_stalled_', ''):40s} {100 * s / tot:6.1f}%")


def launches(path):
    text = open(path).read()
    lines = [l for l in text.splitlines() if l.startswith('"')]
    rows = list(csv.reader(io.StringIO("\n".join(lines))))
    hdr = rows[0]
    ki, mi, vi = hdr.index("Kernel Name"), hdr.index("Metric Name"), hdr.index("Metric Value")
    agg = defaultdict(list)
    for r in rows[1:]:
        if r[mi] == "gpu__time_duration.sum":
            agg[r[ki][:80]].append(float(r[vi].replace(",", "")))
    total = sum(sum(v) for v in agg.values())
    print(f"{'kernel':82s} {'launches':>8s} {'avg':>12s} {'share':>7s}")
    for k, v in sorted(agg.items(), key=lambda kv: -sum(kv[1])):
        print(f"{k:82s} {len(v):8d} {sum(v) / len(v):12.1f} {100 * sum(v) / total:6.1f}%")
    print("(gpu__time_duration.sum per launch; ncu serialises and runs cold-cache, "
          "compare shares, not absolutes; unit as reported by ncu)")


if __name__ == "__main__":
    if sys.argv[1] == "--launches":
        launches(sys.argv[2])
    else:
        report(sys.argv[1])
