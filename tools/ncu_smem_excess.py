"""Shared-memory wavefronts beyond the ideal, per CUDA source line of one kernel.
Usage: python tools/ncu_smem_excess.py report.ncu-rep kernel-regex"""
import csv, io, subprocess, sys
rep, kern = sys.argv[1], sys.argv[2]
txt = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass", "-k", f"regex:{kern}"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(txt)))
fname,hdr="?",None; L=[]
for r in rows:
    if not r: continue
    if r[0]=="File Path": fname=r[1].split('/')[-1]
    elif r[0]=="Line No": hdr=r
    elif hdr and r[0] not in ("","Function Name") and r[2]=="-": L.append((fname,r[0],r[1],r))
def fv(x):
    try: return float(x)
    except: return 0.0
ex=hdr.index("L1 Wavefronts Shared Excessive"); w=hdr.index("L1 Wavefronts Shared"); wi=hdr.index("L1 Wavefronts Shared Ideal")
tot=sum(fv(l[3][ex]) for l in L)
print("excessive total", tot)
for f,ln,src,r in sorted(L,key=lambda l:-fv(l[3][ex]))[:15]:
    print(f"{100*fv(r[ex])/tot:5.1f}% {f}:{ln} wf={fv(r[w]):.3g} ideal={fv(r[wi]):.3g} {src.strip()[:70]}")
