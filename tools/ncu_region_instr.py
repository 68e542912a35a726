"""Instructions executed (all / FP64) and stall-sample share per barrier-delimited SASS region of one kernel.
Usage: python tools/ncu_region_instr.py report.ncu-rep kernel-regex"""
import csv, io, subprocess, sys
from collections import Counter
rep, kern = sys.argv[1], sys.argv[2]
txt = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass", "-k", f"regex:{kern}"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(txt)))
h = rows[1]; data=[r for r in rows[2:] if len(r)>5]
# dedupe: stop at first repeat of address of row 0
a0=data[0][0]
for i in range(1,len(data)):
    if data[i][0]==a0: data=data[:i]; break
def fv(x):
    try: return float(x)
    except: return 0.0
ie=h.index("Instructions Executed")
stall_cols = [i for i, x in enumerate(h) if x.startswith("stall_") and "Not Issued" not in x]
tot=sum(fv(r[c]) for r in data for c in stall_cols)
totie=sum(fv(r[ie]) for r in data)
s0=0
for i,r in enumerate(data):
    s=r[1].strip()
    if ("BAR." in s) or "EXIT" in s or i==len(data)-1:
        seg=data[s0:i+1]
        smp=sum(fv(x[c]) for x in seg for c in stall_cols)
        ni=sum(fv(x[ie]) for x in seg)
        fp=sum(fv(x[ie]) for x in seg if x[1].split()[0].lstrip('@!P0123456789 ').split('.')[0] in ('DFMA','DADD','DMUL') or any(k in x[1] for k in (' DFMA',' DADD',' DMUL')))
        if ni>0.002*totie or smp>0.005*tot:
            print(f"[{s0:5d}-{i:5d}] samp {100*smp/tot:5.1f}% instr {ni:.3g} ({100*ni/totie:4.1f}%) fp64 {fp:.3g}  end: {s[:45]}")
        s0=i+1
print("total instr", totie)
