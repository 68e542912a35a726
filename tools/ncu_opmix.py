"""Executed-instruction histogram by SASS opcode (ncu source page).
Usage: python tools/ncu_opmix.py report.ncu-rep kernel-regex [points]"""
import collections
import csv
import io
import subprocess
import sys

rep, kern = sys.argv[1], sys.argv[2]
npts = float(sys.argv[3]) if len(sys.argv) > 3 else 256.0 ** 3
txt = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "-k", f"regex:{kern}"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(txt)))
starts = [i for i, r in enumerate(rows) if r and r[0] == "Address"]
h = rows[starts[0]]
data = [r for r in rows[starts[0] + 1:(starts[1] - 1 if len(starts) > 1 else None)] if len(r) > 5]
src, ex = h.index("Source"), h.index("Thread Instructions Executed")
hist = collections.Counter()
for r in data:
    s = r[src].strip()
    if s.startswith("@"):
        s = s.split(None, 1)[1] if " " in s else s
    op = s.split()[0] if s else "?"
    try:
        hist[op] += float(r[ex])
    except ValueError:
        pass
tot = sum(hist.values())
print(f"total thread-instructions per point: {tot / npts:.1f}")
for op, n in hist.most_common(30):
    print(f"  {op:28s} {n / npts:8.1f}  {100 * n / tot:5.1f}%")
