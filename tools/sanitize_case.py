"""Small cases for compute-sanitizer: every order, ragged grids, RK3 + Euler,
residual, diagnostics, loopback slabs.  Usage: python tools/sanitize_case.py"""
import math
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1609_01277_b200 as osbli  # noqa: E402
from inputs import TGV_PHYS, perturbed_tgv  # noqa: E402

for order in (2, 4, 6, 8, 10, 12):
    for shape in ((37, 19, 14), (16, 16, 16)):
        dx = 2 * math.pi / max(shape)
        Q = perturbed_tgv(*shape, dx=dx, amp=0.02, kmax=2)
        for scheme in (0, 1):
            s = osbli.Solver(*shape, order, dx, 1e-3, scheme=scheme, **TGV_PHYS)
            s.set_state(Q)
            s.step(1)
            s.residual()
            s.diagnostics()
            s.close()
    g = osbli.LoopbackGroup(20, 12, 4 * order, order, 0.3, 1e-3, 2, **TGV_PHYS)
    g.set_state(perturbed_tgv(20, 12, 4 * order, dx=0.3, amp=0.02, kmax=2))
    g.step(1)
    g.slabs[0].diagnostics()
    g.close()
print("sanitize cases done")
