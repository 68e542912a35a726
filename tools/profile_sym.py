import math, os, sys
sys.path.insert(0, os.getcwd())
import paper_1609_01277_b200 as osbli
from inputs import TGV_PHYS, tgv
n = 256
s = osbli.Solver(n, n, n, 12, 2 * math.pi / n, 3.385e-3 * 64 / n, **TGV_PHYS)
for d in range(3):
    s.set_boundary(d, osbli.OSBLI_BC_SYMMETRY)
s.set_state(tgv(n, n, n))
s.step(1)
s.sync()
print("ok")
