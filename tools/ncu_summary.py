#!/usr/bin/env python
"""Summarise ncu outputs into text files under profiles/.

  python tools/ncu_summary.py full  REPORT.ncu-rep  OUT.txt   # --set full capture
  python tools/ncu_summary.py launches LAUNCHES.csv OUT.txt   # gpu__time_duration list
"""
import csv
import subprocess
import sys
from collections import defaultdict

KEYS = [
    "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
    "dram__bytes_read.sum.per_second", "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
    "sm__throughput.avg.pct_of_peak_sustained_elapsed",
    "smsp__issue_active.avg.pct_of_peak_sustained_active", "smsp__inst_executed.sum",
    "launch__registers_per_thread", "launch__grid_size", "launch__block_size",
    "launch__shared_mem_per_block_dynamic", "sm__warps_active.avg.pct_of_peak_sustained_active",
    "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum", "sm__cycles_elapsed.avg.per_second",
]


def full(rep, out):
    raw = subprocess.check_output(["ncu", "-i", rep, "--page", "raw", "--csv"], text=True,
                                  stderr=subprocess.DEVNULL)
    rows = list(csv.reader(raw.splitlines()))
    hdr, units = rows[0], rows[1]
    lines = []
    for r in rows[2:]:
        d = dict(zip(hdr, r))
        u = dict(zip(hdr, units))
        lines.append(f"kernel: {d.get('Kernel Name', '?')[:160]}")
        for k in KEYS:
            if k in d:
                lines.append(f"  {k:60s} {d[k]:>20s} {u.get(k, '')}")
        stalls = [(k, d[k]) for k in hdr if k.startswith("smsp__pcsamp_warps_issue_stalled_")
                  and not k.endswith("_not_issued")]
        stalls = sorted(((float(v.replace(",", "")) if v else 0.0, k) for k, v in stalls), reverse=True)
        lines.append("  stall samples (top):")
        for v, k in stalls[:8]:
            lines.append(f"    {k.replace('smsp__pcsamp_warps_issue_stalled_', ''):28s} {v:10.0f}")
    open(out, "w").write("\n".join(lines) + "\n")
    print("\n".join(lines))


def launches(path, out):
    rows = list(csv.reader(open(path)))
    start = next(i for i, r in enumerate(rows) if r and r[0] == "ID")
    hdr = rows[start]
    iname, ival = hdr.index("Kernel Name"), hdr.index("Metric Value")
    agg = defaultdict(list)
    order = []
    for r in rows[start + 1:]:
        if len(r) > ival and r[ival]:
            nm = r[iname].split("(")[0][:90]
            if nm not in agg:
                order.append(nm)
            agg[nm].append(float(r[ival].replace(",", "")))
    tot = sum(sum(v) for v in agg.values())
    lines = [f"{'launches':>8s} {'avg_us':>10s} {'total_us':>12s} {'share':>7s}  kernel"]
    for nm in order:
        v = agg[nm]
        lines.append(f"{len(v):8d} {sum(v) / len(v) / 1e3:10.2f} {sum(v) / 1e3:12.1f} "
                     f"{100 * sum(v) / tot:6.1f}%  {nm}")
    open(out, "w").write("\n".join(lines) + "\n")
    print("\n".join(lines))


if __name__ == "__main__":
    {"full": full, "launches": launches}[sys.argv[1]](sys.argv[2], sys.argv[3])
