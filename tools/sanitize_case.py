"""Cases for compute-sanitizer (run with OSBLI_NO_SPLIT=1 so that small grids keep
the production launch shape: 8-plane xy-pass segments with their cross-plane
buffer reuse and group hand-offs, z-pass pencils that advance their ring over
several chunks).  Every order, ragged grids, Euler / RK3 / two-register RK3,
residual, standalone and fused diagnostics, symmetry and the equation variants,
loopback slabs in the three schedules.
Usage: OSBLI_NO_SPLIT=1 python tools/sanitize_case.py [quick]"""
import math
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1609_01277_b200 as osbli  # noqa: E402
from inputs import TGV_PHYS, perturbed_tgv  # noqa: E402

quick = len(sys.argv) > 1 and sys.argv[1] == "quick"
orders = (4, 12) if quick else (2, 4, 6, 8, 10, 12)
for order in orders:
    # 40 x 36: 2 x 3 ragged xy tiles; 72 planes: 9 xy segments of 8, 3 z chunks (ring advance)
    for shape in ((40, 36, 72),) if quick else ((40, 36, 72), (37, 19, 14)):
        dx = 2 * math.pi / max(shape)
        Q = perturbed_tgv(*shape, dx=dx, amp=0.02, kmax=2)
        for scheme in (0, 1, 2):
            s = osbli.Solver(*shape, order, dx, 1e-3, scheme=scheme, **TGV_PHYS)
            s.set_state(Q)
            s.step(1)
            s.residual()
            s.diagnostics()
            s.step_diag(2)
            s.close()
        if order in (4, 12):
            for var in ("sym", "visc", "cons"):
                s = osbli.Solver(*shape, order, dx, 1e-3, **TGV_PHYS)
                if var == "sym":
                    for d in range(3):
                        s.set_boundary(d, osbli.OSBLI_BC_SYMMETRY)
                elif var == "visc":
                    s.set_viscosity(osbli.OSBLI_VISC_SUTHERLAND, 110.4 / 288.0)
                else:
                    s.set_energy_form(osbli.OSBLI_ENERGY_CONSERVATIVE)
                s.set_state(Q)
                s.step(1)
                s.residual()
                s.step_diag(1)
                s.close()
    for sched in (0, 1, 2):
        g = osbli.LoopbackGroup(20, 12, 8 * order, order, 0.3, 1e-3, 2, **TGV_PHYS)
        for sl in g.slabs:
            sl.set_slab_schedule(sched)
        g.set_state(perturbed_tgv(20, 12, 8 * order, dx=0.3, amp=0.02, kmax=2))
        g.step(1)
        g.slabs[0].diagnostics()
        g.close()
    s = osbli.Solver(24, 20, 8 * order, order, 0.3, 1e-3, rank=0, nranks=1,
                     unique_id=osbli.nccl_unique_id(), **TGV_PHYS)
    s.set_slab_schedule(2)
    s.set_state(perturbed_tgv(24, 20, 8 * order, dx=0.3, amp=0.02, kmax=2))
    s.step_diag(2)
    s.step(1)
    s.diagnostics()
    s.close()
print("sanitize cases done")
