"""Minimal driver for ncu: TGV n^3 at the given order, a few RK3 steps.
Usage: python tools/profile_step.py [n] [order] [steps]"""
import math
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_1609_01277_b200 as osbli  # noqa: E402
from inputs import TGV_PHYS, tgv  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 256
order = int(sys.argv[2]) if len(sys.argv) > 2 else 12
steps = int(sys.argv[3]) if len(sys.argv) > 3 else 2
s = osbli.Solver(n, n, n, order, 2 * math.pi / n, 3.385e-3 * 64 / n, **TGV_PHYS)
s.set_state(tgv(n, n, n))
s.step(steps)
s.sync()
print("ok", s.diagnostics())
