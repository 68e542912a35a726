"""BASELINE configs[1]: TGV 64^3, 4th order, RK3, Re = 1600, t = 0..20 on one
B200 — the kinetic-energy / enstrophy / dissipation history (the
paper's figures of it are missing from the text).
Usage: python tools/tgv_history.py [out.csv] [n] [order] [every]"""
import math
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

import paper_1609_01277_b200 as osbli  # noqa: E402
from inputs import TGV_PHYS, tgv  # noqa: E402

out = sys.argv[1] if len(sys.argv) > 1 else "profiles/r2_tgv64_o4_history.csv"
n = int(sys.argv[2]) if len(sys.argv) > 2 else 64
order = int(sys.argv[3]) if len(sys.argv) > 3 else 4
every = int(sys.argv[4]) if len(sys.argv) > 4 else 10
dt = 3.385e-3 * 64 / n
nsteps = int(math.ceil(20.0 / dt))
s = osbli.Solver(n, n, n, order, 2 * math.pi / n, dt, **TGV_PHYS)
s.set_state(tgv(n, n, n))
rows = []
t0 = time.perf_counter()
# diagnostics of every step's input state, fused into the step (osbli_step_diag),
# then the final state's through osbli_diagnostics
for d in s.step_diag(nsteps):
    if d.step % every == 0:
        rows.append((d.step, d.t, d.kinetic_energy, d.enstrophy, d.dissipation))
d = s.diagnostics()
rows.append((d.step, d.t, d.kinetic_energy, d.enstrophy, d.dissipation))
el = time.perf_counter() - t0
a = np.array(rows)
# -dE_k/dt by central differences of the series (SURVEY §8(c) row 12 cross-check)
dek = np.full(len(a), np.nan)
dek[1:-1] = -(a[2:, 2] - a[:-2, 2]) / (a[2:, 1] - a[:-2, 1])
with open(out, "w") as f:
    f.write(f"# TGV {n}^3 order {order} RK3 Re=1600 M=0.1 dt={dt} steps={nsteps}; "
            f"one B200, {el:.1f} s wall with the diagnostics of every step (fused); rows every {every} steps\n")
    f.write("step,t,kinetic_energy,enstrophy,dissipation,minus_dEk_dt\n")
    for r, g in zip(a, dek):
        f.write(f"{int(r[0])},{r[1]:.6f},{r[2]:.15e},{r[3]:.15e},{r[4]:.15e},{g:.6e}\n")
ipk = int(np.argmax(a[:, 3]))
print(f"wrote {out}: {len(a)} rows, E_k(0) = {a[0, 2]:.15f}, enstrophy peak {a[ipk, 3]:.4f} at "
      f"t = {a[ipk, 1]:.2f}, E_k(20) = {a[-1, 2]:.5f}, {el:.1f} s")
