"""Brief summary of an ncu --set full report: headline counters, stall breakdown, instruction mix
by opcode, and the hottest SASS lines (by stall samples).  python tools/ncu_brief.py report.ncu-rep"""
import csv
import io
import subprocess
import sys
from collections import Counter

KEYS = ["gpu__time_duration.sum", "smsp__issue_active.avg.pct_of_peak_sustained_active",
        "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_tensor_subpipe_dmma.avg.pct_of_peak_sustained_active",
        "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed",
        "dram__throughput.avg.pct_of_peak_sustained_elapsed", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread",
        "launch__grid_size", "launch__block_size", "smsp__inst_executed.sum"]


def main(path):
    raw = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    hdr, units, vals = rows[0], rows[1], rows[2]
    d = dict(zip(hdr, vals))
    u = dict(zip(hdr, units))
    out = [f"ncu report: {path}", f"kernel: {d.get('Kernel Name')}"]
    for k in KEYS:
        if k in d:
            out.append(f"  {k:80s} {d[k]} {u.get(k, '')}")
    st = {k: float(v) for k, v in d.items() if k.startswith("smsp__pcsamp_warps_issue_stalled_")
          and not k.endswith("not_issued") and v.replace(".", "", 1).isdigit()}
    tot = sum(st.values()) or 1.0
    out.append("  warp stall samples (share):")
    for k, v in sorted(st.items(), key=lambda kv: -kv[1])[:10]:
        out.append(f"    {100 * v / tot:5.1f}%  {k.replace('smsp__pcsamp_warps_issue_stalled_', '')}")
    src = subprocess.run(["ncu", "-i", path, "--page", "source", "--csv"], capture_output=True, text=True).stdout
    srows = list(csv.reader(io.StringIO(src)))
    h = srows[1]
    ie, sc, ss = h.index("Instructions Executed"), h.index("Source"), h.index("Warp Stall Sampling (All Samples)")
    ops, tot_i = Counter(), 0.0
    lines = []
    for r in srows[2:]:
        try:
            n, s = float(r[ie]), float(r[ss])
        except (ValueError, IndexError):
            continue
        t = r[sc].strip()
        toks = t.replace("@", "").split()
        if not toks:
            continue
        op = (toks[1] if t.startswith("@") and len(toks) > 1 else toks[0]).split(".")[0]
        ops[op] += n
        tot_i += n
        lines.append((s, n, t))
    out.append(f"  executed warp instructions {tot_i:.4g}; by opcode:")
    out.append("    " + ", ".join(f"{op} {100 * n / tot_i:.1f}%" for op, n in ops.most_common(16)))
    out.append("  hottest SASS (stall samples, executions):")
    for s, n, t in sorted(lines, key=lambda x: -x[0])[:12]:
        out.append(f"    {s:8.0f} {n:10.3g}  {t[:90]}")
    print("\n".join(out))


if __name__ == "__main__":
    main(sys.argv[1])
