"""Per-source-line executed instructions and stall samples of one kernel in an ncu report, joined
with nvdisasm line info of the cubin it ran (tools/ncu_lines.py report.ncu-rep object.o kernel_mangled)."""
import csv
import io
import os
import re
import subprocess
import sys
import tempfile
from collections import defaultdict


def main(rep, obj, fn, top=45):
    with tempfile.TemporaryDirectory() as d:
        subprocess.run(["cuobjdump", "-xelf", "all", os.path.abspath(obj)], cwd=d, capture_output=True)
        cub = [f for f in os.listdir(d) if f.endswith(".cubin")][0]
        sass = subprocess.run(["nvdisasm", "-g", os.path.join(d, cub)], capture_output=True, text=True).stdout.split("\n")
    start = next(i for i, l in enumerate(sass) if l.startswith(".text." + fn + ":"))
    cur, a2l = None, {}
    for l in sass[start + 1:]:
        if l.startswith("//--------------------- .text."):
            break
        m = re.match(r'\s*//## File "([^"]+)", line (\d+)', l)
        if m:
            cur = (os.path.basename(m.group(1)), int(m.group(2)))
            continue
        m = re.match(r'\s*/\*([0-9a-f]{4,})\*/\s+', l)
        if m and cur:
            a2l[int(m.group(1), 16)] = cur
    raw = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                         capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    h = rows[1]
    ia, ie, ist = h.index("Address"), h.index("Instructions Executed"), h.index("Warp Stall Sampling (All Samples)")
    base = int(rows[2][ia], 16)
    agg = defaultdict(lambda: [0.0, 0.0])
    tot = [0.0, 0.0]
    for r in rows[2:]:
        try:
            a, n, s = int(r[ia], 16) - base, float(r[ie]), float(r[ist])
        except (ValueError, IndexError):
            continue
        k = a2l.get(a, ("?", 0))
        agg[k][0] += n
        agg[k][1] += s
        tot[0] += n
        tot[1] += s
    srcs = {}
    print(f"{rep}: {tot[0]:.4g} warp instructions")
    for k, (n, s) in sorted(agg.items(), key=lambda kv: -kv[1][0])[:top]:
        path = os.path.join(os.path.dirname(os.path.abspath(obj)), "..", k[0]) if False else None
        txt = ""
        for cand in ("paper_2111_14317_b200/csrc/" + k[0],):
            if os.path.exists(cand):
                srcs.setdefault(cand, open(cand).read().split("\n"))
                txt = srcs[cand][k[1] - 1].strip()[:80] if k[1] > 0 else ""
        print(f"{100 * n / tot[0]:5.1f}% inst {100 * s / tot[1]:5.1f}% stall  {k[0]}:{k[1]}  {txt}")


if __name__ == "__main__":
    main(*sys.argv[1:4])
