"""Where the no_instruction (instruction-fetch) stalls of one kernel land: per SASS address window of
a report's source page, with the executed instructions and the source line of the window start.
    python tools/ncu_noinst.py report.ncu-rep [window_instructions]"""
import csv
import io
import subprocess
import sys


def main(rep, win=64):
    src = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                         capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(src)))
    h = rows[1]
    ia, isrc, iex, ino, iall = (h.index("Address"), h.index("Source"), h.index("Instructions Executed"),
                                h.index("stall_no_inst"), h.index("Warp Stall Sampling (All Samples)"))
    recs = []
    for r in rows[2:]:
        try:
            recs.append((int(r[ia], 16), r[isrc].strip(), float(r[iex] or 0), float(r[ino] or 0), float(r[iall] or 0)))
        except (ValueError, IndexError):
            pass
    recs.sort()
    base = recs[0][0]
    tot_no = sum(x[3] for x in recs) or 1
    tot_all = sum(x[4] for x in recs) or 1
    print(f"{rep}: {len(recs)} instructions ({len(recs) * 16 / 1024:.0f} KB), no_inst {100 * tot_no / tot_all:.1f}% of samples")
    out = []
    for i in range(0, len(recs), win):
        w = recs[i:i + win]
        no = sum(x[3] for x in w)
        ex = sum(x[2] for x in w)
        out.append((no, i, ex, w[0][1]))
    for no, i, ex, s0 in sorted(out, reverse=True)[:25]:
        print(f"  +0x{(recs[i][0] - base):05x} ({i:5d}) no_inst {100 * no / tot_no:5.1f}%  exec {ex:.3g}  {s0[:60]}")


if __name__ == "__main__":
    main(sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else 64)
