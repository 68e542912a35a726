"""Stall samples per CUDA source line of one kernel (ncu source page, cuda+sass view).
Usage: python tools/ncu_lines.py report.ncu-rep kernel-regex [top]"""
import csv
import io
import subprocess
import sys
from collections import Counter

rep, kern = sys.argv[1], sys.argv[2]
top = int(sys.argv[3]) if len(sys.argv) > 3 else 40
txt = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass",
                      "-k", f"regex:{kern}"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(txt)))
fname, hdr = "?", None
lines = []
for r in rows:
    if not r:
        continue
    if r[0] == "File Path":
        fname = r[1].split("/")[-1]
    elif r[0] == "Line No":
        hdr = r
    elif hdr and r[0] not in ("", "Function Name") and r[2] == "-":
        lines.append((fname, r[0], r[1], r))


def fv(x):
    try:
        return float(x)
    except ValueError:
        return 0.0


si = hdr.index("Warp Stall Sampling (All Samples)")
ie = hdr.index("Instructions Executed")
stall_cols = [i for i, x in enumerate(hdr) if x.startswith("stall_") and "Not Issued" not in x]
tot = sum(fv(l[3][si]) for l in lines)
print(f"total samples {tot:.0f}")
for f, ln, src, r in sorted(lines, key=lambda l: -fv(l[3][si]))[:top]:
    st = Counter({hdr[c][6:]: fv(r[c]) for c in stall_cols})
    s = sum(st.values()) or 1
    brk = ", ".join(f"{k}={100 * v / s:.0f}" for k, v in st.most_common(4))
    print(f"{100 * fv(r[si]) / tot:5.1f}% {f}:{ln:>4} ie={fv(r[ie]):.2e} [{brk}] {src.strip()[:60]}")
