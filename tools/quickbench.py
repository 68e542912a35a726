"""Quick device-timed throughput of a config (no JSON contract): n order steps."""
import math
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_1609_01277_b200 as osbli  # noqa: E402
from inputs import TGV_PHYS, tgv  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 256
order = int(sys.argv[2]) if len(sys.argv) > 2 else 12
steps = int(sys.argv[3]) if len(sys.argv) > 3 else 20
scheme = int(sys.argv[4]) if len(sys.argv) > 4 else 1
variant = sys.argv[5] if len(sys.argv) > 5 else ""  # "v": Sutherland mu(T), "c": conservative work
s = osbli.Solver(n, n, n, order, 2 * math.pi / n, 3.385e-3 * 64 / n, scheme=scheme, **TGV_PHYS)
if "v" in variant:
    s.set_viscosity(osbli.OSBLI_VISC_SUTHERLAND, 110.4 / 288.0)
if "c" in variant:
    s.set_energy_form(osbli.OSBLI_ENERGY_CONSERVATIVE)
st = torch.cuda.Stream()
s.set_stream(st.cuda_stream)
s.set_state(tgv(n, n, n))
s.step(3)
s.sync()
s.set_kernel_timing(True)
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record(st)
s.step(steps)
e1.record(st)
torch.cuda.synchronize()
ms = e0.elapsed_time(e1)
z, x, nz_, nx_ = s.kernel_timing()
print(f"{os.environ.get('OSBLI_LIB', 'default')}: n={n} o={order} scheme={scheme}{' ' + variant if variant else ''}: {ms / steps:.3f} ms/step "
      f"{n ** 3 * steps / ms / 1e6:.3f} G pt-steps/s  zpass {z / nz_:.3f} ms  xypass {x / nx_:.3f} ms")
