"""Experiment timing (no kernel timing events): n order steps -> ms/step.
Used for the z/xy overlap measurement of DESIGN.md §5b with OSBLI_ZP_GRID (a
persistent z-pass grid, -DOSBLI_ZP_PERSIST=1 builds) and the OSBLI_EXP_CONC switch
of run_stage (commit 032e30c, removed since; results were wrong by design)."""
import math
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_1609_01277_b200 as osbli  # noqa: E402
from inputs import TGV_PHYS, tgv  # noqa: E402

n, order, steps = (int(a) for a in sys.argv[1:4])
s = osbli.Solver(n, n, n, order, 2 * math.pi / n, 3.385e-3 * 64 / n, scheme=1, **TGV_PHYS)
st = torch.cuda.Stream()
s.set_stream(st.cuda_stream)
s.set_state(tgv(n, n, n))
s.step(3)
s.sync()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record(st)
s.step(steps)
e1.record(st)
torch.cuda.synchronize()
ms = e0.elapsed_time(e1)
tag = " ".join(f"{k}={os.environ[k]}" for k in ("OSBLI_LIB", "OSBLI_EXP_CONC", "OSBLI_ZP_GRID") if k in os.environ)
print(f"{tag}: n={n} o={order}: {ms / steps:.3f} ms/step")
