"""Locate GPU-vs-oracle residual differences (planes, rows, columns)."""
import math
import sys

import os
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

from oracle import core as oracle
import paper_1609_01277_b200 as osbli
from inputs import TGV_PHYS, perturbed_tgv

shape = tuple(int(v) for v in sys.argv[1].split(",")) if len(sys.argv) > 1 else (40, 36, 33)
order = int(sys.argv[2]) if len(sys.argv) > 2 else 2
dx = 2 * math.pi / max(shape)
Q = perturbed_tgv(*shape, dx=dx, amp=0.02)
s = osbli.Solver(*shape, order, dx, 1e-3, **TGV_PHYS)
s.set_state(Q)
R = s.residual()
Ro = oracle.residual(oracle.OracleParams(*shape, order, dx, **TGV_PHYS), Q)
d = np.abs(R - Ro).max(axis=0) / np.abs(Ro).max()
bad = d > 1e-11
print("bad points", bad.sum(), "of", bad.size)
zs, ys, xs = np.nonzero(bad)
print("z planes", sorted(set(zs.tolist()))[:40])
print("y rows", sorted(set(ys.tolist()))[:40])
print("x cols", sorted(set(xs.tolist()))[:40])
for rep in range(3):
    R2 = s.residual()
    print("repeat identical:", np.array_equal(R, R2))
