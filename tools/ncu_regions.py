"""Stall-sample share per barrier-delimited region of a kernel (ncu source page).
Usage: python tools/ncu_regions.py report.ncu-rep kernel-regex"""
import csv
import io
import subprocess
import sys

rep, kern = sys.argv[1], sys.argv[2]
txt = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "-k", f"regex:{kern}"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(txt)))
starts = [i for i, r in enumerate(rows) if r and r[0] == "Address"]
h = rows[starts[0]]
data = [r for r in rows[starts[0] + 1:(starts[1] - 1 if len(starts) > 1 else None)] if len(r) > 5]
si, src = h.index("Warp Stall Sampling (All Samples)"), h.index("Source")


def iv(x):
    try:
        return int(x)
    except ValueError:
        return 0


tot = sum(iv(r[si]) for r in data)
acc, start = 0, 0
for i, r in enumerate(data):
    acc += iv(r[si])
    if "BAR.SYNC" in r[src] or "EXIT" in r[src] or i == len(data) - 1:
        print(f"region {start:5d}-{i:5d}: {100.0 * acc / tot:5.1f}%  ends with {r[src].strip()[:30]}")
        acc, start = 0, i + 1
top = sorted(range(len(data)), key=lambda i: -iv(data[i][si]))[:12]
for i in sorted(top):
    print(f"  {i:5d} {100.0 * iv(data[i][si]) / tot:4.1f}% {data[i][src].strip()[:70]}")
