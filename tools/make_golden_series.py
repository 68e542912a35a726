"""Write tests/golden/tgv64_o4_rk3_series.csv with the ORACLE's diagnostics series.

Calls only oracle/ (and the shared input generator).  BASELINE configs[1]:
TGV 64^3, 4th order, RK3, Re=1600, dt = 3.385e-3.  Columns:
step, t, kinetic_energy, enstrophy, dissipation (17 significant digits).
Usage: python tools/make_golden_series.py [nsteps]
"""
import math
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

from inputs import TGV_PHYS, tgv  # noqa: E402
from oracle import core  # noqa: E402

n = 64
nsteps = int(sys.argv[1]) if len(sys.argv) > 1 else 1000
dt = 3.385e-3
p = core.OracleParams(n, n, n, 4, 2 * math.pi / n, dt=dt, **TGV_PHYS)
series, _ = core.run_series(p, tgv(n, n, n), 1, nsteps)
out = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests", "golden",
                   "tgv64_o4_rk3_series.csv")
with open(out, "w") as f:
    f.write("# oracle diagnostics, TGV 64^3 order 4 RK3 dt=3.385e-3 Re=1600 (tools/make_golden_series.py)\n")
    f.write("step,t,kinetic_energy,enstrophy,dissipation\n")
    for s in range(nsteps + 1):
        f.write("%d,%.17g,%.17g,%.17g,%.17g\n" % (s, s * dt, *series[s]))
print("wrote", out)
