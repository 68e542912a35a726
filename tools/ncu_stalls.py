"""Stall reasons and instruction mix per SASS address range of one kernel (ncu source page).
Usage: python tools/ncu_stalls.py report.ncu-rep kernel-regex [lo-hi ...]
Without ranges: the ranges between BAR.SYNC/EXIT instructions."""
import csv
import io
import re
import subprocess
import sys
from collections import Counter

rep, kern = sys.argv[1], sys.argv[2]
txt = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "-k", f"regex:{kern}"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(txt)))
starts = [i for i, r in enumerate(rows) if r and r[0] == "Address"]
h = rows[starts[0]]
data = [r for r in rows[starts[0] + 1:(starts[1] - 1 if len(starts) > 1 else None)] if len(r) > 5]
src = h.index("Source")
ie = h.index("Instructions Executed")
stall_cols = [i for i, x in enumerate(h) if x.startswith("stall_") and "Not Issued" not in x]


def iv(x):
    try:
        return float(x)
    except ValueError:
        return 0.0


if len(sys.argv) > 3:
    ranges = [tuple(int(v) for v in a.split("-")) for a in sys.argv[3:]]
else:
    ranges, s0 = [], 0
    for i, r in enumerate(data):
        if "BAR.SYNC" in r[src] or "EXIT" in r[src] or i == len(data) - 1:
            ranges.append((s0, i))
            s0 = i + 1
tot = sum(iv(r[c]) for r in data for c in stall_cols)
for lo, hi in ranges:
    seg = data[lo:hi + 1]
    st = Counter()
    ops = Counter()
    for r in seg:
        for c in stall_cols:
            st[h[c][6:]] += iv(r[c])
        op = r[src].strip().split()
        if op:
            o = op[0] if not op[0].startswith("@") else (op[1] if len(op) > 1 else op[0])
            ops[o.split(".")[0]] += iv(r[ie])
    s = sum(st.values())
    if s < 0.01 * tot:
        continue
    ni = sum(ops.values())
    print(f"[{lo}-{hi}] {100 * s / tot:5.1f}% of samples; instr executed {ni:.3g}")
    print("   stalls:", ", ".join(f"{k}={100 * v / s:.0f}%" for k, v in st.most_common(7)))
    print("   ops:", ", ".join(f"{k}={100 * v / max(ni, 1):.0f}%" for k, v in ops.most_common(9)))
