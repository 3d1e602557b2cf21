#!/usr/bin/env python
"""Summarise an ncu report (full set) or a launch-list CSV into a small text file for profiles/.

    python tools/ncu_summary.py report.ncu-rep [out.txt]
    python tools/ncu_summary.py --launches launches.csv [out.txt]
"""
import csv
import io
import subprocess
import sys
from collections import Counter, defaultdict

KEYS = [
    "gpu__time_duration.sum", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
    "dram__bytes_read.sum", "dram__bytes_write.sum", "dram__throughput.avg.pct_of_peak_sustained_elapsed",
    "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_tensor_subpipe_dmma.avg.pct_of_peak_sustained_active",
    "sm__pipe_tensor_cycles_active_realtime.avg.pct_of_peak_sustained_elapsed",
    "smsp__sass_thread_inst_executed_op_dfma_pred_on.sum", "smsp__sass_thread_inst_executed_op_dmul_pred_on.sum",
    "smsp__sass_thread_inst_executed_op_dadd_pred_on.sum",
    "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread",
    "launch__occupancy_limit_registers", "smsp__issue_active.avg.pct_of_peak_sustained_active",
    "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed",
    "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum", "launch__grid_size", "launch__block_size",
]


def full(path, out):
    raw = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    hdr, units, vals = rows[0], rows[1], rows[2:]
    lines = [f"ncu report: {path}"]
    for v in vals:
        d = dict(zip(hdr, v))
        u = dict(zip(hdr, units))
        lines.append(f"kernel: {d.get('Kernel Name', '?')}")
        for k in KEYS:
            for h in hdr:
                if h == k:
                    lines.append(f"  {k:75s} {d[h]} {u[h]}")
        stalls = [(float(d[h]), h) for h in hdr if "pcsamp_warps_issue_stalled" in h
                  and not h.endswith("not_issued") and d[h] not in ("", "n/a")]
        tot = sum(s for s, _ in stalls) or 1.0
        lines.append("  warp stall samples (share):")
        for s, h in sorted(stalls, reverse=True)[:10]:
            lines.append(f"    {100 * s / tot:5.1f}%  {h.replace('smsp__pcsamp_warps_issue_stalled_', '')}")
    text = "\n".join(lines) + "\n"
    open(out, "w").write(text) if out else sys.stdout.write(text)


def launches(path, out):
    rows = [r for r in csv.reader(open(path)) if len(r) > 10]
    hdr = rows[0]
    ki, vi = hdr.index("Kernel Name"), hdr.index("Metric Value")
    t = defaultdict(float)
    c = Counter()
    for r in rows[1:]:
        name = r[ki].split("(")[0]
        t[name] += float(r[vi])
        c[name] += 1
    tot = sum(t.values())
    lines = [f"launch list: {path} (ncu gpu__time_duration.sum, cold-cache, serialised)"]
    for name, v in sorted(t.items(), key=lambda x: -x[1]):
        lines.append(f"  {100 * v / tot:6.2f}%  {c[name]:4d} launches  {v / c[name] / 1e3:10.1f} us/launch  {name}")
    text = "\n".join(lines) + "\n"
    open(out, "w").write(text) if out else sys.stdout.write(text)


if __name__ == "__main__":
    if sys.argv[1] == "--launches":
        launches(sys.argv[2], sys.argv[3] if len(sys.argv) > 3 else None)
    else:
        full(sys.argv[1], sys.argv[2] if len(sys.argv) > 2 else None)
